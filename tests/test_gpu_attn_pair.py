"""K4 kernel schedules (Plan(attn_kernel=...), include/moddit.h mod_attn_kernel) against the fp64 oracle:
the default kernel, the round-1 split-KV kernel ("splitkv") and the paired-query-block kernel ("pair";
SURVEY §8(f) f4).  (The round-1 CTA-pair kernel with M = 256 cta_group::2 MMAs, "pair2", measured 25 %
slower and was retired in round 2.)

The pair kernel walks the merged index list of query blocks 2p and 2p+1 and shares each K/V tile
between them, so its masks are chosen to exercise every shape of that merge: lists that coincide,
alternate, are disjoint (long one-sided stretches that force the early PV drain), are empty on one or
both sides, an odd number of query blocks (a pair with no second block) and a ragged last block.
Tolerances as in test_gpu_parity.py (BASELINE.json north_star): O max-abs <= 2e-2, mean-abs <= 2e-3,
lse <= 5e-3 abs, against the plain masked softmax attention of Eq. 1 in fp64.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn
from gpu_helpers import masks_to_csr, olayout

pytestmark = pytest.mark.gpu

ODD = syn.Workload("odd-n", 1, 2, 128, 0, 3, 20, 19, 128)            # N=1140: n=9 (odd), ragged tail 116
COG_SMALL = syn.Workload("cog-small", 1, 2, 64, 226, 3, 30, 45, 128)  # N=4276, D=64, n=34, ragged 52
SMALL_PREFIX = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)


@pytest.fixture(scope="module")
def M():
    import paper_2601_11641_b200 as m
    return m


KERNELS = ["default", "splitkv", "pair", "wide"]


@pytest.fixture(params=KERNELS)
def kernel(request):
    return request.param


def _check(o, lse, masks, q, k, v, L):
    orf, lrf = O.masked_attention(q.cpu(), k.cpu(), v.cpu(), masks, L)
    og, lg = o.double().cpu().numpy(), lse.double().cpu().numpy()
    err = np.abs(og - orf)
    assert err.max() <= 2e-2, err.max()
    assert err.mean() <= 2e-3, err.mean()
    fin = np.isfinite(lrf)
    assert np.array_equal(np.isfinite(lg), fin)
    assert np.abs(lg[fin] - lrf[fin]).max() <= 5e-3
    # rows of an empty list: O = 0, lse = -inf (reading Z15)
    for b, h, i in zip(*np.nonzero(~masks.any(-1))):
        lo, hi = L.block_range(int(i))
        assert torch.all(o[b, h, lo:hi] == 0) and torch.all(torch.isneginf(lse[b, h, lo:hi]))


def _adversarial(L, heads, seed):
    """Row pairs (2p, 2p+1) cycling through the merge cases of the pair kernel."""
    rng = np.random.default_rng(seed)
    n = L.n
    m = np.zeros((1, heads, n, n), dtype=bool)
    for h in range(heads):
        for p in range(0, n, 2):
            case = (p // 2 + h) % 7
            a = np.zeros(n, dtype=bool)
            b = np.zeros(n, dtype=bool)
            if case == 0:                      # identical lists
                a[:] = rng.random(n) < 0.4
                b[:] = a
            elif case == 1:                    # strictly alternating columns
                a[0::2] = True
                b[1::2] = True
            elif case == 2:                    # disjoint halves: long one-sided stretches
                a[: n // 2] = True
                b[n // 2:] = True
            elif case == 3:                    # A full, B a single block
                a[:] = True
                b[rng.integers(0, n)] = True
            elif case == 4:                    # A empty, B random
                b[:] = rng.random(n) < 0.5
            elif case == 5:                    # both empty
                pass
            else:                              # diagonal bands shifted by one (the MOD-DiT C patterns)
                for d in (-5, 0, 3, 7):
                    if 0 <= p + d < n:
                        a[p + d] = True
                    if 0 <= p + 1 + d < n:
                        b[p + 1 + d] = True
                b[0] = a[0] = True             # a shared vertical column
            m[0, h, p] = a
            if p + 1 < n:
                m[0, h, p + 1] = b
    return m


@pytest.mark.parametrize("w", [ODD, COG_SMALL, SMALL_PREFIX], ids=lambda w: w.name)
def test_pair_merge_cases(M, kernel, w):
    L = olayout(w)
    P = M.Plan(w, attn_kernel=kernel)
    q, k, v = syn.family_r(w, seed=707, device="cuda")
    masks = _adversarial(L, w.heads, 3)
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    _check(o, lse, masks, q, k, v, L)


@pytest.mark.parametrize("density", [0.15, 0.6, 1.0])
def test_pair_random_density(M, kernel, density):
    w = ODD
    L = olayout(w)
    P = M.Plan(w, attn_kernel=kernel)
    q, k, v = syn.family_r(w, seed=708, device="cuda")
    rng = np.random.default_rng(9)
    masks = rng.random((1, w.heads, L.n, L.n)) < density
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    _check(o, lse, masks, q, k, v, L)


def test_variants_agree_on_structured_masks(M):
    """Every schedule on MOD-DiT pattern masks at a CogVideoX-like shape (D=64, text prefix)."""
    w = COG_SMALL
    L = olayout(w)
    q, k, v = syn.family_s(w, device="cuda")
    rng = np.random.default_rng(12)
    masks = np.zeros((1, w.heads, L.n, L.n), dtype=bool)
    for h in range(w.heads):
        sel = O.select_patterns(rng.standard_normal(3 * L.n - 1), L.n, O.SELECT_TOPK, 12)
        masks[0, h] = O.block_mask(sel, rng.random(L.frames) < 0.7, L, True)
    rp, ci = masks_to_csr(masks)
    res = {kern: M.Plan(w, attn_kernel=kern).block_sparse_attn_fwd(q, k, v, rp, ci) for kern in KERNELS}
    torch.cuda.synchronize()
    for kern in res:
        _check(*res[kern], masks, q, k, v, L)
    # different accumulation orders (split-KV merge vs one accumulator): close, not bitwise
    for kern in res:
        assert (res[kern][0].float() - res["default"][0].float()).abs().max().item() <= 2e-2


@pytest.mark.parametrize("kern", KERNELS)
def test_variant_deterministic(M, kern):
    w = COG_SMALL
    L = olayout(w)
    P = M.Plan(w, attn_kernel=kern)
    q, k, v = syn.family_r(w, device="cuda")
    masks = _adversarial(L, w.heads, 4)
    rp, ci = masks_to_csr(masks)
    o1, l1 = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    o2, l2 = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("kern", ["default", "splitkv"])
@pytest.mark.parametrize("w", [syn.TINY, syn.Workload("b64-d128", 1, 2, 128, 0, 2, 10, 13, 64)], ids=lambda w: w.name)
def test_block64(M, kern, w):
    """64-token blocks (the tiny config, D = 64; and D = 128): more S buffers, half-width softmax rows."""
    L = olayout(w)
    P = M.Plan(w, attn_kernel=kern)
    q, k, v = syn.family_r(w, seed=709, device="cuda")
    rng = np.random.default_rng(10)
    masks = rng.random((1, w.heads, L.n, L.n)) < 0.5
    masks[0, 0, 1] = False
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    _check(o, lse, masks, q, k, v, L)


@pytest.mark.parametrize("kern", KERNELS)
def test_row_maximum_jumps(M, kern):
    """Key blocks scaled by 1..60 in list order make the row maximum jump by up to ~100 (log2 units)
    between blocks -- beyond the default kernel's lazy reference bound (2^20), so its exchange / redo /
    O-rescale path runs -- and also fall back to small values afterwards (stale reference max)."""
    w = ODD
    L = olayout(w)
    P = M.Plan(w, attn_kernel=kern)
    q, k, v = syn.family_r(w, seed=711, device="cuda")
    k = k.clone()
    scales = [1.0, 3.0, 12.0, 0.5, 25.0, 60.0, 2.0, 40.0, 1.0]
    for j in range(L.n):
        lo, hi = L.block_range(j)
        k[:, :, lo:hi] = (k[:, :, lo:hi].float() * scales[j % len(scales)]).to(torch.bfloat16)
    rng = np.random.default_rng(13)
    masks = rng.random((1, w.heads, L.n, L.n)) < 0.7
    masks[0, 0, 0] = True
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    _check(o, lse, masks, q, k, v, L)


@pytest.mark.parametrize("kern", KERNELS)
@pytest.mark.parametrize("stride", [3, 13])
def test_runs_of_empty_rows(M, kern, stride):
    """Only every stride-th query block has a list (long runs of empty rows: the persistent schedule's
    item ring then runs more than its depth ahead of the softmax and must keep issuing the V loads it
    owes); the listed rows are long and the empty ones must still come out as O = 0, lse = -inf (Z15)."""
    w = COG_SMALL
    L = olayout(w)
    P = M.Plan(w, attn_kernel=kern)
    q, k, v = syn.family_r(w, seed=715, device="cuda")
    rng = np.random.default_rng(stride)
    masks = np.zeros((1, w.heads, L.n, L.n), dtype=bool)
    for h in range(w.heads):
        for i in range(h, L.n, stride):
            masks[0, h, i] = rng.random(L.n) < 0.5
            masks[0, h, i, i] = True
    rp, ci = masks_to_csr(masks)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    torch.cuda.synchronize()
    _check(o, lse, masks, q, k, v, L)
