"""Algorithm 1 on the GPU (paper_2601_11641_b200.Schedule) against the oracle schedule, tiny config."""
import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn
from gpu_helpers import csr_to_masks, olayout

pytestmark = pytest.mark.gpu


def test_schedule_matches_oracle_tiny():
    import paper_2601_11641_b200 as M
    from paper_2601_11641_b200.schedule import Schedule
    w = syn.TINY
    L = olayout(w)
    K = 3
    P = M.Plan(w, top_k=K)
    sch = Schedule(P, T=50, m=12, dt=10)
    osch = O.OracleSchedule(L, T=50, m=12, dt=10, top_k=K)
    agree = 0
    for t in range(1, 51):
        q, k, v = syn.family_s(w, step=t, device="cuda")
        o, lse = sch.step(t, q, k, v)
        torch.cuda.synchronize()
        got = csr_to_masks(*sch.last_mask, L.n)
        ref_mask, _ = osch.step(t, q.cpu(), k.cpu(), v.cpu(), compute_attention=False)
        agree += int(np.array_equal(got, ref_mask))
        # the attention itself is checked against the oracle under the mask the GPU used
        o_ref, l_ref = O.masked_attention(q.cpu(), k.cpu(), v.cpu(), got, L)
        err = np.abs(o.double().cpu().numpy() - o_ref)
        assert err.max() <= 2e-2 and err.mean() <= 2e-3
    assert agree >= 48          # masks bit-exact except possibly inside the Top-K tie band (Z14)
    assert sch.state.t_prev == 32 and sch.state.t_curr == 42


def test_schedule_exact_statistic_matches_oracle_tiny():
    """Alg. 1 with the paper's own Eq. 2 statistic on the GPU vs the oracle schedule."""
    import paper_2601_11641_b200 as M
    from paper_2601_11641_b200.schedule import Schedule
    w = syn.TINY
    L = olayout(w)
    K = 3
    P = M.Plan(w, top_k=K, masked_renorm=False)
    sch = Schedule(P, T=30, m=12, dt=5, stat="exact", eta=1e-4)
    osch = O.OracleSchedule(L, T=30, m=12, dt=5, top_k=K, masked_renorm=False, stat="exact", eta=1e-4)
    agree = 0
    for t in range(1, 31):
        q, k, v = syn.family_s(w, step=t, device="cuda")
        o, lse = sch.step(t, q, k, v)
        torch.cuda.synchronize()
        got = csr_to_masks(*sch.last_mask, L.n)
        ref_mask, _ = osch.step(t, q.cpu(), k.cpu(), v.cpu(), compute_attention=False)
        agree += int(np.array_equal(got, ref_mask))
        o_ref, _ = O.masked_attention(q.cpu(), k.cpu(), v.cpu(), got, L)
        err = np.abs(o.double().cpu().numpy() - o_ref)
        assert err.max() <= 2e-2 and err.mean() <= 2e-3
    assert agree >= 27


def test_schedule_q8_same_masks_as_bf16():
    """Alg. 1 with the quantized sparse attention: the pooled statistic does not depend on the
    attention's precision, so every step's mask is bit-identical to the bf16 schedule's; the outputs
    agree to the quantization error (DESIGN.md parity bar for f2)."""
    import paper_2601_11641_b200 as M
    from paper_2601_11641_b200.schedule import Schedule
    w = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)
    P = M.Plan(w, top_k=6)
    a = Schedule(P, T=30, m=12, dt=10)
    b = Schedule(P, T=30, m=12, dt=10, precision="q8")
    for t in range(1, 31):
        q, k, v = syn.family_s(w, step=t, device="cuda")
        oa, _ = a.step(t, q, k, v)
        oa = oa.clone()
        ob, _ = b.step(t, q, k, v)
        (ra, ca), (rb, cb) = a.last_mask, b.last_mask
        assert torch.equal(ra, rb)                                          # col_idx: used prefix only
        for h in range(w.heads):
            nnz = int(ra[0, h, -1])
            assert torch.equal(ca[0, h, :nnz], cb[0, h, :nnz])
        d = (oa.float() - ob.float()).abs()
        if t <= 12:
            assert d.max().item() == 0.0                                  # warm-up: same bf16 kernel
        else:
            assert d.max().item() <= 0.1 and d.mean().item() <= 6e-3
    with pytest.raises(ValueError, match="stat='pooled'"):
        Schedule(P, precision="q8", stat="exact")


def test_schedule_sdpa_warmup_same_masks():
    """warmup_attention='sdpa' (library dense kernel for the full-attention warm-up, as the paper's FA2)
    leaves the pooled statistics -- hence every mask -- unchanged, and its warm-up output matches K4's."""
    import paper_2601_11641_b200 as M
    from paper_2601_11641_b200.schedule import Schedule
    w = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)
    P = M.Plan(w, top_k=6)
    a = Schedule(P, T=20, m=12, dt=10)
    b = Schedule(P, T=20, m=12, dt=10, warmup_attention="sdpa")
    for t in range(1, 21):
        q, k, v = syn.family_s(w, step=t, device="cuda")
        oa, _ = a.step(t, q, k, v)
        oa = oa.clone()
        ob, _ = b.step(t, q, k, v)
        (ra, ca), (rb, cb) = a.last_mask, b.last_mask
        assert torch.equal(ra, rb)
        for h in range(w.heads):
            nnz = int(ra[0, h, -1])
            assert torch.equal(ca[0, h, :nnz], cb[0, h, :nnz])
        d = (oa.float() - ob.float()).abs()
        assert d.max().item() <= 2e-2
    with pytest.raises(ValueError, match="stat='pooled'"):
        Schedule(P, warmup_attention="sdpa", stat="exact")
