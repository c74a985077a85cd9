"""Algorithm 1 on the GPU (paper_2601_11641_b200.Schedule) against the oracle schedule, tiny config."""
import numpy as np
import pytest
import torch

import oracle as O
import synthetic as syn
from gpu_helpers import csr_to_masks, olayout

pytestmark = pytest.mark.gpu


def _state(x_prev, x_curr, t_prev, t_curr, keep):
    f = lambda x: x.double().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64)
    return f(x_prev), f(x_curr), t_prev, t_curr, np.asarray(keep.cpu().numpy() if isinstance(keep, torch.Tensor) else keep)


def _check_step_mask(got, g_state, o_state, L, K, rel_tol):
    """One sparse step of Alg. 1: the GPU mask must be (a) exactly the oracle's predict + select + mask
    applied to the GPU's own intensities (integer work bit-exact given X), and (b) the oracle's own mask
    except for patterns inside the Top-K tie band (reading Z14): every pattern selected by one side only
    has an oracle key within 2*delta of the oracle's K-th key, delta = max |key_gpu - key_oracle|, and
    delta itself is within the numerical bound rel_tol * max|key|.  Returns True when the masks agree."""
    xp_g, xc_g, tp, tc, keep_g = g_state
    xp_o, xc_o, tp_o, tc_o, keep_o = o_state
    assert (tp, tc) == (tp_o, tc_o)
    t = got.t
    ref_from_gpu_x = O.predict_block_mask(xp_g, xc_g, tp, tc, t, keep_g, L, O.SELECT_TOPK, K, 0.0, True)
    assert np.array_equal(got.mask, ref_from_gpu_x)                       # (a)
    o_ = 3 * L.n - 1
    e_o = np.minimum(xp_o[..., o_:], xc_o[..., o_:])
    e_d = np.maximum(np.abs(xp_g - xp_o)[..., o_:], np.abs(xc_g - xc_o)[..., o_:])
    assert np.all((keep_g == keep_o) | (np.abs(e_o) <= 2 * e_d))          # keep flips only at tau_e = 0
    kg = O.pattern_keys(O.extrapolate(xp_g, xc_g, tp, tc, t), L)
    ko = O.pattern_keys(O.extrapolate(xp_o, xc_o, tp, tc, t), L)
    same = True
    for b in range(L.batch):
        for h in range(L.heads):
            delta = np.abs(kg[b, h] - ko[b, h]).max()
            assert delta <= rel_tol * np.abs(ko[b, h]).max(), (t, h, delta)
            MAX_REL[0] = max(MAX_REL[0], delta / np.abs(ko[b, h]).max())
            sg = O.select_patterns(kg[b, h], L.n, O.SELECT_TOPK, K)
            so = O.select_patterns(ko[b, h], L.n, O.SELECT_TOPK, K)
            if np.array_equal(sg, so):
                continue
            same = False
            kth = np.sort(ko[b, h])[::-1][K - 1]
            for pidx in np.nonzero(sg ^ so)[0]:
                assert abs(ko[b, h, pidx] - kth) <= 2 * delta, (t, h, pidx)   # (b): inside the tie band
    return same


MAX_REL = [0.0]


class _Got:
    def __init__(self, t, mask):
        self.t, self.mask = t, mask


def _run_schedule_vs_oracle(w, K, T, m, dt, stat, rel_tol, renorm=True, drift=0.0):
    import paper_2601_11641_b200 as M
    from paper_2601_11641_b200.schedule import Schedule
    L = olayout(w)
    P = M.Plan(w, top_k=K, masked_renorm=renorm)
    sch = Schedule(P, T=T, m=m, dt=dt, stat=stat, eta=1e-4)
    osch = O.OracleSchedule(L, T=T, m=m, dt=dt, top_k=K, masked_renorm=renorm, stat=stat, eta=1e-4)
    agree = steps = 0
    for t in range(1, T + 1):
        q, k, v = syn.family_s(w, step=t, device="cuda", drift=drift, steps_total=T)
        if t > m:
            S = sch.state
            g_state = _state(S.x_prev, S.x_curr, S.t_prev, S.t_curr, S.keep)
            o_state = _state(osch.x_prev, osch.x_curr, osch.t_prev, osch.t_curr, osch.keep)
        o, lse = sch.step(t, q, k, v)
        torch.cuda.synchronize()
        got = csr_to_masks(*sch.last_mask, L.n)
        if t > m:
            steps += 1
            agree += _check_step_mask(_Got(t, got), g_state, o_state, L, K, rel_tol)
        else:
            assert got.all()
        # the oracle follows the GPU's mask, so that a tie-band difference at one step does not
        # compound through Eq. 5 into later states (each step is checked on its own)
        osch.step(t, q.cpu(), k.cpu(), v.cpu(), mask_override=got, compute_attention=False)
        # the attention itself is checked against the oracle under the mask the GPU used
        o_ref, l_ref = O.masked_attention(q.cpu(), k.cpu(), v.cpu(), got, L)
        err = np.abs(o.double().cpu().numpy() - o_ref)
        assert err.max() <= 2e-2 and err.mean() <= 2e-3
    return sch, agree, steps


def test_schedule_matches_oracle_tiny():
    # K1's bar is 1e-3 relative on W (fp32 pooled scores); the fit and the Eq. 6/7 extrapolation (up to
    # 21x at t - t_c = 10 over a one-step first window) carry it into the keys
    sch, agree, steps = _run_schedule_vs_oracle(syn.TINY, 3, 50, 12, 10, "pooled", 2e-2)
    print(f"tiny: {agree}/{steps} steps with identical masks, max key delta {MAX_REL[0]:.2e} relative")
    assert steps == 38
    assert sch.state.t_prev == 32 and sch.state.t_curr == 42


def test_schedule_matches_oracle_prefix_layout():
    """Alg. 1 on a ragged prefix layout (D = 128, 20x19 frames, 40 prefix tokens), pooled statistic."""
    w = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)
    sch, agree, steps = _run_schedule_vs_oracle(w, 6, 34, 12, 10, "pooled", 2e-2)
    print(f"prefix: {agree}/{steps} steps with identical masks, max key delta {MAX_REL[0]:.2e} relative")
    assert steps == 22


def test_schedule_drifting_trajectories_prefix_layout():
    """Alg. 1 over Family S with drifting pattern strengths (§4.3: intensities evolve
    piecewise-linearly, which Eq. 6/7 extrapolate and Eq. 5 reconstructs): the masks now change over
    the sparse steps, and every step still matches the oracle up to the tie band."""
    w = syn.Workload("small-prefix", 1, 3, 128, 40, 3, 20, 19, 128)
    sch, agree, steps = _run_schedule_vs_oracle(w, 6, 42, 12, 10, "pooled", 2e-2, drift=0.8)
    print(f"drift: {agree}/{steps} steps with identical masks, max key delta {MAX_REL[0]:.2e} relative")
    assert steps == 30


def test_schedule_exact_statistic_matches_oracle_tiny():
    """Alg. 1 with the paper's own Eq. 2 statistic on the GPU vs the oracle schedule.  The
    GPU thresholds with K4's fp32 lse, the oracle with fp64: a few counts at eta may move, so the key
    bound is looser (1e-1 relative) while every mask difference must still sit inside the tie band."""
    sch, agree, steps = _run_schedule_vs_oracle(syn.TINY, 3, 30, 12, 5, "exact", 1e-1, renorm=False)
    print(f"exact: {agree}/{steps} steps with identical masks, max key delta {MAX_REL[0]:.2e} relative")


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


def test_schedule_k1_side_stream_bitwise_equal_to_serial():
    """K1 on the side stream beside K4 (the default) changes only the order of independent work: every
    step's O, lse and mask, and the final history / intensities, equal the serial schedule's bit for bit."""
    import paper_2601_11641_b200 as M
    w = syn.Workload("sched-prefix", 1, 3, 128, 40, 3, 20, 19, 128)
    q, k, v = syn.family_s(w, device="cuda")
    from paper_2601_11641_b200.schedule import Schedule
    scheds = [Schedule(M.Plan(w, top_k=6, tau_e=0.0), T=30, m=6, dt=5, overlap_k1=ov) for ov in (True, False)]
    for t in range(1, 31):
        qt, kt, vt = syn.family_s(w, step=t, device="cuda") if t > 1 else (q, k, v)
        res = [s_.step(t, qt, kt, vt) for s_ in scheds]
        torch.cuda.synchronize()
        assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1]), t
        (rpa, cia), (rpb, cib) = scheds[0].last_mask, scheds[1].last_mask
        assert torch.equal(rpa, rpb), t
        nnz = rpa[..., -1].cpu()
        for h in range(w.heads):   # the index lists (the capacity beyond nnz is unspecified)
            assert torch.equal(cia[0, h, : nnz[0, h]], cib[0, h, : nnz[0, h]]), (t, h)
    sa, sb = scheds[0].state, scheds[1].state
    assert torch.equal(sa.hist, sb.hist) and torch.equal(sa.x_prev, sb.x_prev) and torch.equal(sa.x_curr, sb.x_curr)
