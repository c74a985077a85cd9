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
