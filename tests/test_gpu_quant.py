"""GPU parity of the quantized sparse attention (reading Z30) through the C ABI.

* codes and scales (integer decisions taken in fp32 on both sides): bit-exact vs oracle/quant.py
* O vs the fp64 attention over the dequantized Q^, K^, V^: the GPU also rounds P to e4m3 (3 mantissa
  bits, relative rounding error <= 2^-4), which the oracle does not model; the bar (DESIGN.md
  "Parity") is max-abs <= 0.08 and mean-abs <= 4e-3 on unit-variance inputs, lse <= 2e-3 abs
  (lse is summed from the fp32 probabilities)."""
import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn
from gpu_helpers import masks_to_csr, olayout

pytestmark = pytest.mark.gpu

SMALL = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)      # N=1180, ragged tail 28
MAX_ABS, MEAN_ABS, LSE_ABS = 0.08, 4e-3, 2e-3


@pytest.fixture(scope="module")
def M():
    import paper_2601_11641_b200 as m
    return m


def _e4m3_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.float8_e4m3fn).to(torch.float64).numpy()


@pytest.mark.parametrize("family", ["R", "S"])
def test_quantize_codes_bit_exact(M, family):
    w = SMALL
    L = olayout(w)
    P = M.Plan(w)
    q, k, v = (syn.family_r(w, device="cuda") if family == "R" else syn.family_s(w, step=3, device="cuda"))
    qb = P.quantize_qkv(q, k, v)
    qb2 = P.quantize_qkv(q, k, v)
    torch.cuda.synchronize()
    V = {key: t.cpu().numpy() for key, t in P.quant_views(qb).items()}
    V2 = {key: t.cpu().numpy() for key, t in P.quant_views(qb2).items()}
    assert all(np.array_equal(V[key], V2[key]) for key in V)                 # deterministic
    Np = V["vt8"].shape[-1]
    for h in range(w.heads):
        Qh, Kh, Vh = (t[0, h].float().cpu().numpy() for t in (q, k, v))
        qc, qs = O.quantize_int8_blocks(Qh, L)
        kc, ks = O.quantize_int8_blocks(Kh, L)
        vv, vs = O.quantize_e4m3_channels(Vh)
        assert np.array_equal(V["q8"][0, h], qc) and np.array_equal(V["q_scale"][0, h], qs)
        assert np.array_equal(V["k8"][0, h], kc) and np.array_equal(V["k_scale"][0, h], ks)
        assert np.array_equal(V["v_scale"][0, h], vs)
        vt = _e4m3_bits_to_f64(V["vt8"][0, h])                              # [D, Np]
        assert np.array_equal(vt[:, :L.N].T, vv)
        assert np.all(vt[:, L.N:Np] == 0)


def _masks(w, L, seed, density=0.4):
    rng = np.random.default_rng(seed)
    m = rng.random((w.batch, w.heads, L.n, L.n)) < density
    m |= np.eye(L.n, dtype=bool)
    return m


@pytest.mark.parametrize("family", ["R", "S"])
def test_attention_q8_parity(M, family):
    w = SMALL
    L = olayout(w)
    P = M.Plan(w)
    q, k, v = (syn.family_r(w, device="cuda") if family == "R" else syn.family_s(w, step=5, device="cuda"))
    masks = _masks(w, L, 7)
    masks[0, 1, 2, :] = False                                               # an empty row (no diag)
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd_q8(P.quantize_qkv(q, k, v), rp, ci)
    torch.cuda.synchronize()
    og, lg = o.float().cpu().numpy(), lse.cpu().numpy()
    errs = []
    for h in range(w.heads):
        Qh, Kh, Vh = (t[0, h].float().cpu().numpy() for t in (q, k, v))
        outs, lses = O.quantized_attention_rows(Qh, Kh, Vh, masks[0, h], L, range(L.n))
        for i, (orf, lrf) in enumerate(zip(outs, lses)):
            lo, hi = L.block_range(i)
            if not masks[0, h, i].any():
                assert np.all(og[0, h, lo:hi] == 0) and np.all(np.isneginf(lg[0, h, lo:hi]))
                continue
            d = np.abs(og[0, h, lo:hi] - orf)
            errs.append(d)
            assert np.max(np.abs(lg[0, h, lo:hi] - lrf)) <= LSE_ABS
    d = np.concatenate([e.ravel() for e in errs])
    assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS, (d.max(), d.mean())


def test_attention_q8_close_to_bf16_path(M):
    """Same mask: the quantized and the bf16 kernels agree to the quantization error."""
    w = SMALL
    L = olayout(w)
    P = M.Plan(w)
    q, k, v = syn.family_r(w, device="cuda")
    rp, ci = masks_to_csr(_masks(w, L, 9, 0.6))
    o8, l8 = P.block_sparse_attn_fwd_q8(P.quantize_qkv(q, k, v), rp, ci)
    ob, lb = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    d = (o8.float() - ob.float()).abs()
    assert d.max().item() <= 0.1 and d.mean().item() <= 6e-3
    assert (l8 - lb).abs().max().item() <= 0.05


def test_quant_unsupported_layouts(M):
    P = M.Plan(syn.TINY)                                                    # head_dim 64, block 64
    assert M.lib.mod_quant_buffer_bytes(P.handle) == 0
    with pytest.raises(M.ModditError, match="head_dim=128, block=128"):
        P.quant_buffer()


@pytest.mark.parametrize("w", [syn.HUNYUAN, syn.WAN], ids=lambda w: w.name)
def test_attention_q8_full_size_sampled(M, w):
    """Full BASELINE shapes (D = 128), structured masks; codes of the sampled heads bit-exact, O of
    sampled query blocks (first, last ragged, heaviest row, random) within the f2 bar."""
    L = olayout(w)
    P = M.Plan(w)
    q, k, v = syn.family_s(w, step=7, device="cuda")
    rng = np.random.default_rng(81)
    masks = np.zeros((1, w.heads, L.n, L.n), dtype=bool)
    for h in range(w.heads):
        sel = O.select_patterns(rng.standard_normal(3 * L.n - 1), L.n, O.SELECT_TOPK, max(4, L.n // 10))
        masks[0, h] = O.block_mask(sel, rng.random(L.frames) < 0.7, L, True)
    rp, ci = masks_to_csr(masks)
    qb = P.quantize_qkv(q, k, v)
    o, lse = P.block_sparse_attn_fwd_q8(qb, rp, ci)
    torch.cuda.synchronize()
    views = P.quant_views(qb)
    errs = []
    for h in (0, w.heads - 1):
        Qh, Kh, Vh = (t[0, h].float().cpu().numpy() for t in (q, k, v))
        qc, qs = O.quantize_int8_blocks(Qh, L)
        assert np.array_equal(views["q8"][0, h].cpu().numpy(), qc)
        assert np.array_equal(views["q_scale"][0, h].cpu().numpy(), qs)
        counts = masks[0, h].sum(1)
        blocks = sorted({0, L.n - 1, int(np.argmax(counts)), int(rng.integers(0, L.n))})
        outs, lses = O.quantized_attention_rows(Qh, Kh, Vh, masks[0, h], L, blocks)
        og, lg = o[0, h].float().cpu().numpy(), lse[0, h].cpu().numpy()
        for i, orf, lrf in zip(blocks, outs, lses):
            lo, hi = L.block_range(i)
            errs.append(np.abs(og[lo:hi] - orf).ravel())
            assert np.max(np.abs(lg[lo:hi] - lrf)) <= LSE_ABS
    d = np.concatenate(errs)
    assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS, (d.max(), d.mean())
