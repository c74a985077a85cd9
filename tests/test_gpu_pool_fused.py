"""K1's block means fused into K4 at a re-estimation step (include/moddit.h mod_block_sparse_attn_fwd_pool +
mod_collect_block_stats_pooled; Alg. 1 P:1006-1013 takes the fresh statistic on the step's own Q, K).

* O and lse of the fused launch are bit-identical to mod_block_sparse_attn_fwd (the attention part of the
  kernel is unchanged);
* W from the fused means is within 1e-3 relative of the fp64 oracle (BASELINE.json north_star "pooled
  scores within 1e-3 relative"), and within 1e-5 relative of the unfused K1 (both are fp32 sums of the same
  bf16 tokens in different orders);
* every query block's means are written, also for rows whose index list is empty (the K_i tile is
  loaded for the pool alone), for ragged last blocks, 64-token blocks and D = 64 / 128; the schedules
  without the fused pool (wide at D = 64, split-KV) run K1's pool kernel after the attention.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn
from gpu_helpers import masks_to_csr, olayout

pytestmark = pytest.mark.gpu

ODD = syn.Workload("odd-n", 1, 2, 128, 0, 3, 20, 19, 128)            # N=1140: n=9, ragged tail 116
COG_SMALL = syn.Workload("cog-small", 1, 2, 64, 226, 3, 30, 45, 128)  # D=64: wide schedule (pool kernel after)
SMALL_PREFIX = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)
B64_D128 = syn.Workload("b64-d128", 1, 2, 128, 0, 2, 10, 13, 64)


@pytest.fixture(scope="module")
def M():
    import paper_2601_11641_b200 as m
    return m


def _masks(L, heads, seed, empty_every=4):
    rng = np.random.default_rng(seed)
    m = rng.random((1, heads, L.n, L.n)) < 0.4
    for h in range(heads):
        for i in range(L.n):
            m[0, h, i, i] = True
        m[0, h, h % empty_every::empty_every] = False   # rows with an empty list (Z15)
    return m


@pytest.mark.parametrize("w", [syn.TINY, ODD, SMALL_PREFIX, B64_D128, COG_SMALL], ids=lambda w: w.name)
@pytest.mark.parametrize("kern", ["default", "splitkv"])
def test_fused_pool_matches_k1_and_oracle(M, w, kern):
    L = olayout(w)
    P = M.Plan(w, attn_kernel=kern)
    q, k, v = syn.family_s(w, device="cuda")
    rp, ci = masks_to_csr(_masks(L, w.heads, 31))
    o0, l0 = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    W0 = P.collect_block_stats(q, k)
    o1, l1 = P.block_sparse_attn_fwd(q, k, v, rp, ci, pool=True)
    W1 = P.collect_block_stats_pooled()
    torch.cuda.synchronize()
    assert torch.equal(o0, o1) and torch.equal(l0, l1)
    ref = O.pooled_block_stats(q.cpu(), k.cpu(), L)
    Wf = W1.double().cpu().numpy()
    assert np.all(np.abs(Wf - ref) <= 1e-3 * ref + 1e-9)
    W0d = W0.double().cpu().numpy()
    assert np.all(np.abs(Wf - W0d) <= 1e-5 * W0d + 1e-12)
    assert np.allclose(Wf.sum(-1), 1.0, atol=1e-5)


def test_fused_pool_stale_workspace_overwritten(M):
    """The fused means overwrite whatever the workspace held (a previous K1 on other tensors)."""
    w = SMALL_PREFIX
    L = olayout(w)
    P = M.Plan(w)
    q, k, v = syn.family_r(w, seed=41, device="cuda")
    q2, k2, _ = syn.family_r(w, seed=42, device="cuda")
    rp, ci = masks_to_csr(_masks(L, w.heads, 32))
    P.collect_block_stats(q2, k2)                   # leaves q2 / k2 means in the workspace
    P.block_sparse_attn_fwd(q, k, v, rp, ci, pool=True)
    W = P.collect_block_stats_pooled()
    torch.cuda.synchronize()
    ref = O.pooled_block_stats(q.cpu(), k.cpu(), L)
    assert np.all(np.abs(W.double().cpu().numpy() - ref) <= 1e-3 * ref + 1e-9)


def test_fused_pool_hunyuan_bench_step(M):
    """At the bench shape (Hunyuan 720p, Family S, the predicted K = 164 mask): O bitwise, W vs unfused K1
    and vs the oracle on sampled heads."""
    w = syn.HUNYUAN
    P = M.Plan(w, top_k=1)
    q1, k1, _ = syn.family_s(w, step=11, device="cuda")
    Wa = P.collect_block_stats(q1, k1)
    del q1, k1
    q, k, v = syn.family_s(w, step=12, device="cuda")
    Wb = P.collect_block_stats(q, k)
    x1, x2 = P.fit_mixture(Wa), P.fit_mixture(Wb)
    rp, ci = P.predict_block_mask(x1, x2, 11, 12, 22, P.keep_frames(x1, x2), top_k=164)
    o0, l0 = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    o1, l1 = P.block_sparse_attn_fwd(q, k, v, rp, ci, pool=True)
    W1 = P.collect_block_stats_pooled()
    torch.cuda.synchronize()
    assert torch.equal(o0, o1) and torch.equal(l0, l1)
    assert torch.all((W1.double() - Wb.double()).abs() <= 1e-5 * Wb.double() + 1e-12)
    Lh = olayout(w.with_heads(1))
    for h in (0, 23):
        ref = O.pooled_block_stats(q[:, h:h + 1].cpu(), k[:, h:h + 1].cpu(), Lh)[0, 0]
        assert np.all(np.abs(W1[0, h].double().cpu().numpy() - ref) <= 1e-3 * ref + 1e-9)
