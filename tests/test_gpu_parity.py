"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star):
  * pooled statistic W: elementwise |dW| <= 1e-3 * W (+1e-9)
  * intensities X (fp64): component orthogonal to the null vector <= 1e-8 relative; the
    null-vector component of the oracle's plain Cholesky carries ~cond(G)*u error (App. B
    P:1254-1258 is evaluated literally there), so the total is checked at 50*cond(G)*u
  * keep flags, CSR row_ptr / col_idx: bit-exact given identical intensities; given identical W,
    bit-exact for every head whose K-th/K+1-th key gap exceeds the tie band (reading Z14)
  * history map: unselected entries bit-identical, selected within 1 fp32 ulp
  * attention O: max-abs <= 2e-2, mean-abs <= 2e-3 vs fp64 on unit-variance bf16 inputs;
    lse <= 5e-3 abs
"""
import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn
from gpu_helpers import csr_rows_sorted_unique, csr_to_masks, masks_to_csr, null_vector_c_d, olayout

pytestmark = pytest.mark.gpu

SMALL_PREFIX = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)     # N=1180, ragged tail 28
COG_SMALL = syn.Workload("cog-small", 1, 2, 64, 226, 3, 30, 45, 128)          # N=4276, D=64, ragged 52
TINY = syn.TINY


@pytest.fixture(scope="module")
def M():
    import paper_2601_11641_b200 as m
    return m


def plan_for(M, w, **kw):
    return M.Plan(w, **kw)


def rel_err(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ------------------------------------------------------------------------------------------ K1
@pytest.mark.parametrize("w", [TINY, SMALL_PREFIX, COG_SMALL, syn.COGVIDEOX], ids=lambda w: w.name)
def test_stats_parity(M, w):
    P = plan_for(M, w)
    q, k, _ = syn.family_r(w, device="cuda")
    W = P.collect_block_stats(q, k)
    torch.cuda.synchronize()
    ref = O.pooled_block_stats(q.cpu(), k.cpu(), olayout(w))
    Wg = W.double().cpu().numpy()
    assert np.all(np.abs(Wg - ref) <= 1e-3 * ref + 1e-9)
    assert np.allclose(Wg.sum(-1), 1.0, atol=1e-5)


def test_stats_parity_hunyuan_sampled_heads(M):
    w = syn.HUNYUAN
    P = plan_for(M, w)
    q, k, _ = syn.family_r(w, device="cuda")
    W = P.collect_block_stats(q, k)
    torch.cuda.synchronize()
    L = olayout(w.with_heads(1))
    for h in (0, 23):
        ref = O.pooled_block_stats(q[:, h:h + 1].cpu(), k[:, h:h + 1].cpu(), L)[0, 0]
        Wg = W[0, h].double().cpu().numpy()
        assert np.all(np.abs(Wg - ref) <= 1e-3 * ref + 1e-9)


def test_stats_structured_family_s(M):
    w = COG_SMALL
    P = plan_for(M, w)
    q, k, _ = syn.family_s(w, device="cuda")
    W = P.collect_block_stats(q, k)
    torch.cuda.synchronize()
    ref = O.pooled_block_stats(q.cpu(), k.cpu(), olayout(w))
    assert np.all(np.abs(W.double().cpu().numpy() - ref) <= 1e-3 * ref + 1e-9)


# ------------------------------------------------------------------------------------------ K2a
def _null_basis(L):
    """Orthonormal basis of null(M): numerically from the closed-form Gram when p is moderate,
    else the always-present (1_C, -1_D, 0_E) direction (nullity is 1 for the video layouts)."""
    if L.p <= 1500:
        ev, Q = np.linalg.eigh(O.gram_closed_form(L, lam=0.0))
        return Q[:, ev < 1e-6 * ev[-1]]
    return null_vector_c_d(L.n, L.p)[:, None]


def _check_x(xg, xr, L, G_cond):
    V = _null_basis(L)
    p = L.p
    for a, b in zip(xg.reshape(-1, p), xr.reshape(-1, p)):
        pa, pb = a - V @ (V.T @ a), b - V @ (V.T @ b)
        assert rel_err(pa, pb) <= 1e-8
        assert rel_err(a, b) <= max(1e-8, 50 * G_cond * np.finfo(float).eps)
        assert np.linalg.norm(V.T @ a) <= 1e-9 * np.linalg.norm(a)   # deflated solve stays in the min-norm gauge


@pytest.mark.parametrize("w", [TINY, SMALL_PREFIX, COG_SMALL, syn.COGVIDEOX], ids=lambda w: w.name)
def test_fit_parity(M, w):
    L = olayout(w)
    P = plan_for(M, w)
    U = syn.random_stats(w.batch, w.heads, L.n, seed=7, device="cuda")
    X, nae = P.fit_mixture(U, want_nae=True)
    torch.cuda.synchronize()
    Un = U.double().cpu().numpy()
    xr = O.fit_mixture(Un, L)
    cond = np.linalg.cond(O.gram_closed_form(L)) if L.p <= 1000 else 6e10
    _check_x(X.cpu().numpy(), xr, L, cond)
    for h in range(min(w.heads, 4)):
        assert abs(nae[0, h].item() - O.nae(Un[0, h], xr[0, h], L)) <= 1e-5


def test_fit_parity_hunyuan(M):
    w = syn.HUNYUAN
    L = olayout(w.with_heads(2))
    P = plan_for(M, w.with_heads(2))
    U = syn.random_stats(1, 2, L.n, seed=8, device="cuda")
    X = P.fit_mixture(U)
    torch.cuda.synchronize()
    xr = O.fit_mixture(U.double().cpu().numpy(), L)
    _check_x(X.cpu().numpy(), xr, L, 6e10)


# ------------------------------------------------------------------------------------------ keep / K2b
@pytest.mark.parametrize("w", [TINY, SMALL_PREFIX, COG_SMALL], ids=lambda w: w.name)
def test_keep_bit_exact(M, w):
    L = olayout(w)
    P = plan_for(M, w, tau_e=0.05)
    xa = syn.random_intensities(w.batch, w.heads, L.p, seed=1, device="cuda") * 0.1
    xb = syn.random_intensities(w.batch, w.heads, L.p, seed=2, device="cuda") * 0.1
    keep = P.keep_frames(xa, xb)
    torch.cuda.synchronize()
    ref = O.keep_frames(xa.cpu().numpy(), xb.cpu().numpy(), L, np.float32(0.05))
    assert np.array_equal(keep.cpu().numpy(), ref)


@pytest.mark.parametrize("w", [TINY, SMALL_PREFIX, COG_SMALL, syn.HUNYUAN.with_heads(3)], ids=lambda w: w.name)
@pytest.mark.parametrize("mode,param", [(0, 0.0), (1, 0.4), (2, 0.6)], ids=["topk", "threshold", "topmass"])
def test_predict_bit_exact_given_x(M, w, mode, param):
    L = olayout(w)
    K = max(1, (3 * L.n - 1) // 7)
    P = plan_for(M, w, top_k=K, select_mode=mode, select_param=param)
    xp = syn.random_intensities(w.batch, w.heads, L.p, seed=3, device="cuda")
    xc = syn.random_intensities(w.batch, w.heads, L.p, seed=4, device="cuda")
    keep = (torch.rand((w.batch, w.heads, w.frames), generator=torch.Generator().manual_seed(5)) < 0.5).to(torch.uint8).cuda()
    rp, ci = P.predict_block_mask(xp, xc, 22, 32, 37, keep)
    torch.cuda.synchronize()
    ref = O.predict_block_mask(xp.cpu().numpy(), xc.cpu().numpy(), 22, 32, 37, keep.cpu().numpy(), L, mode, K,
                               float(np.float32(param)), True)
    got = csr_to_masks(rp, ci, L.n)
    assert csr_rows_sorted_unique(rp, ci, L.n)
    assert np.array_equal(got, ref)
    assert np.array_equal(rp[..., -1].cpu().numpy(), ref.sum((-1, -2)))


@pytest.mark.parametrize("w", [SMALL_PREFIX, syn.HUNYUAN.with_heads(2)], ids=lambda w: w.name)
@pytest.mark.parametrize("K", [1, 7, 100, 10 ** 6])
def test_predict_topk_ties_bit_exact(M, w, K):
    """Top-K with massive exact ties, signed zeros and negative keys (reading Z14: ties by ascending
    pattern id): the GPU's radix select must pick the oracle's set."""
    L = olayout(w)
    P = plan_for(M, w, top_k=K)
    g = torch.Generator().manual_seed(91)
    # intensities on a coarse grid of 5 values (incl. 0 and -0) -> keys repeat across many patterns
    vals = torch.tensor([-1.0, -0.0, 0.0, 0.5, 2.0], dtype=torch.float64)
    xc = vals[torch.randint(0, 5, (w.batch, w.heads, L.p), generator=g)].cuda()
    xp = xc.clone()                      # x_hat = x_curr exactly (zero slope)
    rp, ci = P.predict_block_mask(xp, xc, 11, 12, 13, None)
    torch.cuda.synchronize()
    ref = O.predict_block_mask(xp.cpu().numpy(), xc.cpu().numpy(), 11, 12, 13,
                               np.zeros((w.batch, w.heads, w.frames)), L, O.SELECT_TOPK, K, 0.0, True)
    assert np.array_equal(csr_to_masks(rp, ci, L.n), ref)


def test_predict_without_keep_and_guard(M):
    w = SMALL_PREFIX
    L = olayout(w)
    P = plan_for(M, w, top_k=3, diag_guard=False)
    xp = syn.random_intensities(1, w.heads, L.p, seed=6, device="cuda")
    rp, ci = P.predict_block_mask(xp, xp * 2, 11, 12, 13, None)
    torch.cuda.synchronize()
    ref = O.predict_block_mask(xp.cpu().numpy(), 2 * xp.cpu().numpy(), 11, 12, 13, np.zeros((1, w.heads, w.frames)),
                               L, 0, 3, 0.0, False)
    assert np.array_equal(csr_to_masks(rp, ci, L.n), ref)


def test_dense_mask(M):
    w = COG_SMALL
    P = plan_for(M, w)
    rp, ci = P.dense_mask()
    torch.cuda.synchronize()
    assert csr_to_masks(rp, ci, P.n).all()


@pytest.mark.parametrize("w", [SMALL_PREFIX, COG_SMALL, syn.COGVIDEOX], ids=lambda w: w.name)
def test_fit_then_predict_given_identical_stats(M, w):
    """End to end from identical W: masks bit-exact outside the Top-K tie band (reading Z14)."""
    L = olayout(w)
    K = max(2, (3 * L.n - 1) // 6)
    P = plan_for(M, w, top_k=K)
    U1 = syn.random_stats(w.batch, w.heads, L.n, seed=11, device="cuda")
    U2 = syn.random_stats(w.batch, w.heads, L.n, seed=12, device="cuda")
    X1, X2 = P.fit_mixture(U1), P.fit_mixture(U2)
    rp, ci = P.predict_block_mask(X1, X2, 11, 12, 14, None)
    torch.cuda.synchronize()
    x1 = O.fit_mixture(U1.double().cpu().numpy(), L)
    x2 = O.fit_mixture(U2.double().cpu().numpy(), L)
    ref = O.predict_block_mask(x1, x2, 11, 12, 14, np.zeros((1, w.heads, w.frames)), L, 0, K, 0.0, True)
    got = csr_to_masks(rp, ci, L.n)
    # (a) integer work bit-exact given the GPU's own intensities
    xg1, xg2 = X1.cpu().numpy(), X2.cpu().numpy()
    zero_keep = np.zeros((1, w.heads, w.frames))
    assert np.array_equal(got, O.predict_block_mask(xg1, xg2, 11, 12, 14, zero_keep, L, 0, K, 0.0, True))
    # (b) vs the oracle's own intensities: every differing pattern lies inside the Top-K tie band
    # (reading Z14), i.e. within 2*delta of the oracle's K-th key, delta = max |key_gpu - key_oracle|
    ko = O.pattern_keys(O.extrapolate(x1, x2, 11, 12, 14), L).reshape(-1, 3 * L.n - 1)
    kg = O.pattern_keys(O.extrapolate(xg1, xg2, 11, 12, 14), L).reshape(-1, 3 * L.n - 1)
    same = 0
    # the oracle's literal Cholesky carries ~cond(G)*u along null(M), which moves C keys
    # against D keys; Eq. 6/7 at t = 14 from (11, 12) amplifies X differences by at most 1 + 2*2 = 5
    bound = 5 * 50 * np.linalg.cond(O.gram_closed_form(L)) * np.finfo(float).eps
    for t in range(ko.shape[0]):
        delta = np.abs(kg[t] - ko[t]).max()
        assert delta <= bound * max(np.abs(x1).max(), np.abs(x2).max()), (t, delta)
        so = O.select_patterns(ko[t], L.n, O.SELECT_TOPK, K)
        sg = O.select_patterns(kg[t], L.n, O.SELECT_TOPK, K)
        if np.array_equal(so, sg):
            assert np.array_equal(got.reshape(-1, L.n, L.n)[t], ref.reshape(-1, L.n, L.n)[t])
            same += 1
            continue
        kth = np.sort(ko[t])[::-1][K - 1]
        assert all(abs(ko[t, p_] - kth) <= 2 * delta for p_ in np.nonzero(so ^ sg)[0]), t
    assert same >= 1


# ------------------------------------------------------------------------------------------ K3
@pytest.mark.parametrize("w", [TINY, SMALL_PREFIX, COG_SMALL], ids=lambda w: w.name)
@pytest.mark.parametrize("renorm", [True, False])
def test_update_parity(M, w, renorm):
    L = olayout(w)
    P = plan_for(M, w, masked_renorm=renorm)
    Wf = syn.random_stats(w.batch, w.heads, L.n, seed=21, device="cuda")
    hist = syn.random_stats(w.batch, w.heads, L.n, seed=22, device="cuda")
    rng = np.random.default_rng(23)
    masks = rng.random((w.batch, w.heads, L.n, L.n)) < 0.3
    masks |= np.eye(L.n, dtype=bool)
    rp, ci = masks_to_csr(masks)
    xp = syn.random_intensities(w.batch, w.heads, L.p, seed=24, device="cuda")
    xc = syn.random_intensities(w.batch, w.heads, L.p, seed=25, device="cuda")
    hist0, xc0 = hist.cpu().numpy().copy(), xc.cpu().numpy().copy()
    P.update_online_mask(Wf, rp, ci, hist, xp, xc)
    torch.cuda.synchronize()
    ref_hist = O.reconstruct_history(Wf.double().cpu().numpy(), hist0.astype(np.float64), masks, renorm)
    hg = hist.cpu().numpy()
    assert np.array_equal(hg[~masks], hist0[~masks])                                  # Eq. 5 second branch
    ulp = np.spacing(np.abs(ref_hist[masks]).astype(np.float32))
    assert np.all(np.abs(hg[masks].astype(np.float64) - ref_hist[masks]) <= ulp)      # first branch
    assert np.array_equal(xp.cpu().numpy(), xc0)                                       # roll
    xr = O.fit_mixture(hg.astype(np.float64), L)
    _check_x(xc.cpu().numpy(), xr, L, np.linalg.cond(O.gram_closed_form(L)))


# ------------------------------------------------------------------------------------------ K4
def _attn_check(og, lg, orf, lrf):
    err = np.abs(og - orf)
    assert err.max() <= 2e-2, err.max()
    assert err.mean() <= 2e-3, err.mean()
    fin = np.isfinite(lrf)
    assert np.array_equal(np.isfinite(lg), fin)
    assert np.abs(lg[fin] - lrf[fin]).max() <= 5e-3


def _random_masks(w, L, density, seed):
    rng = np.random.default_rng(seed)
    m = rng.random((w.batch, w.heads, L.n, L.n)) < density
    m |= np.eye(L.n, dtype=bool)
    return m


@pytest.mark.parametrize("w,density", [(TINY, 0.5), (SMALL_PREFIX, 0.4), (COG_SMALL, 0.25)],
                         ids=["tiny", "small-prefix", "cog-small"])
def test_attention_parity_full(M, w, density):
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_r(w, device="cuda")
    masks = _random_masks(w, L, density, 31)
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    orf, lrf = O.masked_attention(q.cpu(), k.cpu(), v.cpu(), masks, L)
    _attn_check(o.double().cpu().numpy(), lse.double().cpu().numpy(), orf, lrf)


def test_attention_dense_mask_equals_dense_attention(M):
    w = TINY
    P = plan_for(M, w)
    q, k, v = syn.family_r(w, seed=99, device="cuda")
    rp, ci = P.dense_mask()
    o, _ = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    ref = O.dense_attention(q.cpu(), k.cpu(), v.cpu())
    err = np.abs(o.double().cpu().numpy() - ref)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3


def test_attention_empty_rows(M):
    w = SMALL_PREFIX
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_r(w, device="cuda")
    masks = _random_masks(w, L, 0.3, 41)
    masks[0, 1, 3, :] = False
    masks[0, 2, L.n - 1, :] = False
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    orf, lrf = O.masked_attention(q.cpu(), k.cpu(), v.cpu(), masks, L)
    _attn_check(o.double().cpu().numpy(), lse.double().cpu().numpy(), orf, lrf)
    lo, hi = L.block_range(3)
    assert torch.all(o[0, 1, lo:hi] == 0) and torch.all(torch.isneginf(lse[0, 1, lo:hi]))


def _structured_masks(L, heads, seed, top_k):
    rng = np.random.default_rng(seed)
    out = np.zeros((1, heads, L.n, L.n), dtype=bool)
    for h in range(heads):
        keys = rng.standard_normal(3 * L.n - 1)
        sel = O.select_patterns(keys, L.n, O.SELECT_TOPK, top_k)
        keep = rng.random(L.frames) < 0.7
        out[0, h] = O.block_mask(sel, keep, L, True)
    return out


@pytest.mark.parametrize("w", [syn.HUNYUAN, syn.WAN, syn.COGVIDEOX], ids=lambda w: w.name)
def test_attention_parity_full_size_sampled(M, w):
    """Full BASELINE shapes in the launch configuration bench.py times; oracle on sampled blocks."""
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_r(w, device="cuda")
    masks = _structured_masks(L, w.heads, 51, top_k=max(4, L.n // 10))
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    Lh = olayout(w.with_heads(1))
    rng = np.random.default_rng(52)
    for h in (0, w.heads - 1):
        qh, kh, vh = q[:, h:h + 1].cpu(), k[:, h:h + 1].cpu(), v[:, h:h + 1].cpu()
        counts = masks[0, h].sum(1)
        blocks = sorted({0, L.n - 1, int(np.argmax(counts)), int(rng.integers(0, L.n))})
        outs, lses = O.masked_attention_rows(qh, kh, vh, masks[0, h], Lh, 0, 0, blocks)
        og = o[0, h].double().cpu().numpy()
        lg = lse[0, h].double().cpu().numpy()
        for i, orf, lrf in zip(blocks, outs, lses):
            lo, hi = L.block_range(i)
            _attn_check(og[lo:hi], lg[lo:hi], orf, lrf)


def _rows_check(P, L, q, k, v, o, lse, masks_h, heads, rng, extra_blocks=()):
    """Oracle O/lse on sampled query blocks (first, ragged last, heaviest row, a random one) per head."""
    Lh = O.make_layout(1, 1, L.head_dim, L.prefix_tokens, L.frames, L.height, L.width, L.block)
    for h in heads:
        qh, kh, vh = q[:, h:h + 1].cpu(), k[:, h:h + 1].cpu(), v[:, h:h + 1].cpu()
        mh = masks_h[h]
        counts = mh.sum(1)
        blocks = sorted({0, L.n - 1, int(np.argmax(counts)), int(rng.integers(0, L.n)), *extra_blocks})
        outs, lses = O.masked_attention_rows(qh, kh, vh, mh, Lh, 0, 0, blocks)
        og = o[0, h].double().cpu().numpy()
        lg = lse[0, h].double().cpu().numpy()
        for i, orf, lrf in zip(blocks, outs, lses):
            lo, hi = L.block_range(i)
            _attn_check(og[lo:hi], lg[lo:hi], orf, lrf)


def test_attention_dense_list_full_size_hunyuan(M):
    """K4 on the all-ones index list at HunyuanVideo 720p (the warm-up's full attention, Alg. 1
    P:992-996), Family S inputs (sink columns, frame structure): sampled rows vs fp64 dense attention."""
    w = syn.HUNYUAN
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_s(w, step=M_STEP, device="cuda")
    rp, ci = P.dense_mask()
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    ones = np.ones((L.n, L.n), dtype=bool)
    _rows_check(P, L, q, k, v, o, lse, {h: ones for h in (0, 13, 23)}, (0, 13, 23), np.random.default_rng(91))


M_STEP = 12


def test_attention_bench_mask_full_size_hunyuan(M):
    """K4 on exactly the workload bench.py times: Family S at HunyuanVideo 720p, the mask the pipeline
    predicts for t_p = 22 from the warm-up fits at t = 11, 12 with K = 164 (87.75 % block sparsity)."""
    w = syn.HUNYUAN
    L = olayout(w)
    P = plan_for(M, w, top_k=1, tau_e=0.0)
    q1, k1, _ = syn.family_s(w, step=M_STEP - 1, device="cuda")
    W1 = P.collect_block_stats(q1, k1)
    del q1, k1
    q, k, v = syn.family_s(w, step=M_STEP, device="cuda")
    W2 = P.collect_block_stats(q, k)
    x1, x2 = P.fit_mixture(W1), P.fit_mixture(W2)
    keep = P.keep_frames(x1, x2)
    rp, ci = P.predict_block_mask(x1, x2, M_STEP - 1, M_STEP, M_STEP + 10, keep, top_k=164)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    rpn, cin = rp.cpu().numpy(), ci.cpu().numpy()
    sparsity = 1.0 - rpn[..., -1].sum() / (w.heads * L.n * L.n)
    assert 0.86 <= sparsity <= 0.89, sparsity
    heads = (0, 7, 16, 23)
    masks_h = {h: O.csr_to_mask(rpn[0, h], cin[0, h], L.n) for h in heads}
    _rows_check(P, L, q, k, v, o, lse, masks_h, heads, np.random.default_rng(92), extra_blocks=(L.n // 2,))


def test_attention_deterministic(M):
    w = COG_SMALL
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_r(w, device="cuda")
    rp, ci = masks_to_csr(_random_masks(w, L, 0.3, 61))
    o1, l1 = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    o2, l2 = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


# ------------------------------------------------------------------------------------------ errors
def test_plan_errors(M):
    with pytest.raises(M.ModditError, match="head_dim=96"):
        M.Plan(dict(batch=1, heads=1, head_dim=96, prefix_tokens=0, frames=1, height=4, width=4, block=128))
    with pytest.raises(M.ModditError, match="top_k=0"):
        M.Plan(TINY, top_k=0)
    P = M.Plan(TINY)
    x = P.empty_x()
    with pytest.raises(M.ModditError, match="zero denominator"):
        P.predict_block_mask(x, x, 5, 5, 6)


# ------------------------------------------------------------------------------------------ f1 EXACT statistic
def _exact_check(Ug, S_ref, q, k, lse32, masks, L, eta):
    """Blocks must agree except for probabilities within the fp32 evaluation band of eta."""
    s = 1.0 / np.sqrt(L.head_dim)
    qn, kn = q.double().cpu().numpy(), k.double().cpu().numpy()
    tb = np.arange(L.N) // L.block
    for b in range(masks.shape[0]):
        for h in range(masks.shape[1]):
            A = s * qn[b, h] @ kn[b, h].T - lse32[b, h][:, None]          # ln P with the kernel's lse
            amb = np.abs(A - np.log(eta)) <= 1e-3                          # fp32 dot products + threshold
            for i in range(L.n):
                ilo, ihi = L.block_range(i)
                for j in np.nonzero(masks[b, h, i])[0]:
                    jlo, jhi = L.block_range(j)
                    nb = amb[ilo:ihi, jlo:jhi].sum()
                    tol = (nb + 0.5) / ((ihi - ilo) * (jhi - jlo))
                    assert abs((-Ug[b, h, i, j]) - S_ref[b, h, i, j]) <= tol, (b, h, i, j)


@pytest.mark.parametrize("w", [TINY, SMALL_PREFIX, COG_SMALL], ids=lambda w: w.name)
def test_exact_sparsity_dense_and_masked(M, w):
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_s(w, device="cuda")
    eta = 1e-4
    # dense (warm-up): lse of the full attention
    ones = np.ones((w.batch, w.heads, L.n, L.n), dtype=bool)
    S_ref, lse_ref = O.exact_sparsity_masked(q.cpu(), k.cpu(), ones, L, eta)
    lse32 = torch.from_numpy(lse_ref.astype(np.float32)).cuda()
    rp, ci = P.dense_mask()
    U = P.collect_exact_sparsity(q, k, lse32, rp, ci, eta)
    torch.cuda.synchronize()
    _exact_check(U.double().cpu().numpy(), S_ref, q, k, lse32.double().cpu().numpy(), ones, L, eta)
    assert np.allclose(S_ref, O.exact_sparsity(q.cpu(), k.cpu(), L, eta))
    # masked (re-estimation step): lse over the kept blocks, unlisted entries untouched
    masks = _random_masks(w, L, 0.3, 71)
    S_m, lse_m = O.exact_sparsity_masked(q.cpu(), k.cpu(), masks, L, eta)
    lse32 = torch.from_numpy(lse_m.astype(np.float32)).cuda()
    rp, ci = masks_to_csr(masks)
    U2 = P.collect_exact_sparsity(q, k, lse32, rp, ci, eta)
    torch.cuda.synchronize()
    U2n = U2.double().cpu().numpy()
    assert np.all(np.isnan(U2n[~masks]))
    _exact_check(U2n, S_m, q, k, lse32.double().cpu().numpy(), masks, L, eta)


def test_exact_sparsity_with_kernel_lse(M):
    """End to end on the GPU: K4's own lse (sparse) feeds the EXACT statistic."""
    w = SMALL_PREFIX
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_s(w, device="cuda")
    masks = _random_masks(w, L, 0.4, 72)
    rp, ci = masks_to_csr(masks)
    _, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    U = P.collect_exact_sparsity(q, k, lse, rp, ci, 1e-4)
    torch.cuda.synchronize()
    S_m, _ = O.exact_sparsity_masked(q.cpu(), k.cpu(), masks, L, 1e-4)
    d = np.abs((-U.double().cpu().numpy()[masks]) - S_m[masks])
    assert d.max() <= 0.02 and d.mean() <= 1e-3      # K4 lse error (<= 5e-3) moves a few threshold decisions


# ------------------------------------------------------------------------------------------ full-size samples
def test_update_parity_hunyuan_sampled_heads(M):
    """K3 at the Hunyuan 720p layout (n = 929, p = 2819): Eq. 5 merge bit-level, refit vs the oracle."""
    w = syn.HUNYUAN.with_heads(2)
    L = olayout(w)
    P = plan_for(M, w)
    Wf = syn.random_stats(w.batch, w.heads, L.n, seed=81, device="cuda")
    hist = syn.random_stats(w.batch, w.heads, L.n, seed=82, device="cuda")
    masks = _structured_masks(L, w.heads, 83, top_k=164)
    rp, ci = masks_to_csr(masks)
    xp = syn.random_intensities(w.batch, w.heads, L.p, seed=84, device="cuda")
    xc = syn.random_intensities(w.batch, w.heads, L.p, seed=85, device="cuda")
    hist0, xc0 = hist.cpu().numpy().copy(), xc.cpu().numpy().copy()
    P.update_online_mask(Wf, rp, ci, hist, xp, xc)
    torch.cuda.synchronize()
    ref_hist = O.reconstruct_history(Wf.double().cpu().numpy(), hist0.astype(np.float64), masks, True)
    hg = hist.cpu().numpy()
    assert np.array_equal(hg[~masks], hist0[~masks])
    ulp = np.spacing(np.abs(ref_hist[masks]).astype(np.float32))
    assert np.all(np.abs(hg[masks].astype(np.float64) - ref_hist[masks]) <= ulp)
    assert np.array_equal(xp.cpu().numpy(), xc0)
    xr = O.fit_mixture(hg.astype(np.float64), L)
    _check_x(xc.cpu().numpy(), xr, L, np.linalg.cond(O.gram_closed_form(L)))


def test_exact_sparsity_hunyuan_sampled_rows(M):
    """f1 EXACT statistic at the Hunyuan 720p layout with K4's own lse, on sampled query blocks."""
    w = syn.HUNYUAN.with_heads(1)
    L = olayout(w)
    P = plan_for(M, w)
    q, k, v = syn.family_s(w, device="cuda")
    masks = _structured_masks(L, 1, 86, top_k=164)
    rp, ci = masks_to_csr(masks)
    _, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    U = P.collect_exact_sparsity(q, k, lse, rp, ci, 1e-4)
    torch.cuda.synchronize()
    Un = U.double().cpu().numpy()[0, 0]
    assert np.all(np.isnan(Un[~masks[0, 0]]))
    rng = np.random.default_rng(87)
    counts = masks[0, 0].sum(1)
    blocks = sorted({0, L.n - 1, int(np.argmax(counts)), int(rng.integers(0, L.n))})
    rows = O.exact_sparsity_masked_rows(q.cpu(), k.cpu(), masks[0, 0], L, 0, 0, blocks, 1e-4)
    for i, (row, lse_ref) in rows.items():
        lo, hi = L.block_range(i)
        assert np.abs(lse[0, 0, lo:hi].double().cpu().numpy() - lse_ref).max() <= 5e-3
        sel = ~np.isnan(row)
        d = np.abs((-Un[i][sel]) - row[sel])
        # K4's lse (<= 5e-3) and fp32 dot products move the few probabilities that sit at eta
        assert d.max() <= 0.02 and d.mean() <= 2e-3, (i, d.max(), d.mean())


# ------------------------------------------------------------------------------------------ App. B solver chain
# Layouts whose frame squares create linear dependencies among the bases that the plan's analytic
# null-space list does not know (sub-block frames at the grid corner): the deflated Gram keeps a pivot of
# order lambda, the Cholesky step is rejected and the chain of App. B must end in the
# pseudo-inverse step.  X must still match the oracle's literal Tikhonov solve off null(M).
DEGENERATE = [syn.Workload("degen-2x48", 1, 2, 64, 0, 2, 1, 48, 64),        # frames [0,0], [0,1]
              syn.Workload("degen-prefix", 1, 2, 64, 10, 4, 2, 20, 64),     # nullity 3, analytic 1
              syn.Workload("degen-6x3x14", 1, 2, 64, 0, 6, 3, 14, 64)]


@pytest.mark.parametrize("w", DEGENERATE, ids=lambda w: w.name)
def test_plan_solver_chain_degenerate_layout(M, w):
    L = olayout(w)
    Mx = O.design_matrix(L)
    nullity = L.p - np.linalg.matrix_rank(Mx)
    P = plan_for(M, w)
    assert P.solver == "pinv", (P.solver, P.min_pivot, P.null_dim)
    assert P.null_dim == nullity
    assert P.min_pivot > 1e-4           # every retained direction is well conditioned after the chain
    U = syn.random_stats(w.batch, w.heads, L.n, seed=17, device="cuda")
    X = P.fit_mixture(U)
    torch.cuda.synchronize()
    xr = O.fit_mixture(U.double().cpu().numpy(), L)
    _check_x(X.cpu().numpy(), xr, L, np.linalg.cond(O.gram_closed_form(L)))
    # the pseudo-inverse solution is the minimum-norm least-squares fit: orthogonal to null(M)
    V = _null_basis(L)
    xg = X.cpu().numpy().reshape(-1, L.p)
    assert np.abs(xg @ V).max() <= 1e-9 * np.abs(xg).max()


@pytest.mark.parametrize("w", [TINY, SMALL_PREFIX, syn.HUNYUAN], ids=lambda w: w.name)
def test_plan_solver_chain_video_layouts_stay_cholesky(M, w):
    P = plan_for(M, w)
    assert P.solver == "cholesky" and P.min_pivot > 1e-4 and P.create_ms > 0


def test_fit_and_update_on_head_slices_of_odd_n(M):
    """K2a / K3 on head slices of a larger stats tensor (the head-chunk pipelines pass views): with odd n
    the slices start at addresses that are not 16-byte aligned; results must equal the contiguous copy's
    bit for bit."""
    w = syn.Workload("odd-n", 1, 3, 64, 0, 4, 9, 16, 64)     # N = 576, n = 9
    L = olayout(w)
    assert L.n % 2 == 1
    P1 = plan_for(M, w.with_heads(1))
    U = syn.random_stats(1, 3, L.n, seed=23, device="cuda")
    for h in range(3):
        xa = P1.fit_mixture(U[:, h:h + 1])
        xb = P1.fit_mixture(U[:, h:h + 1].clone())
        torch.cuda.synchronize()
        assert torch.equal(xa, xb), h
