"""Algorithm 1 oracle driver -- no GPU.  SPEC S:483: with K = the full pattern pool every
mask is all-ones and each step's output equals full attention; updates happen at t_p = m + i*dt."""
import numpy as np

import oracle as O
import synthetic as syn


def test_full_pool_equals_dense_every_step():
    w = syn.TINY
    L = O.make_layout(w.batch, w.heads, w.head_dim, w.prefix_tokens, w.frames, w.height, w.width, w.block)
    sch = O.OracleSchedule(L, T=16, m=4, dt=3, top_k=3 * L.n - 1)
    updates = []
    for t in range(1, 17):
        q, k, v = syn.family_s(w, step=t)
        x_before = None if sch.x_curr is None else sch.x_curr.copy()
        mask, (o, _) = sch.step(t, q, k, v)
        assert mask.all()
        assert np.max(np.abs(o - O.dense_attention(q, k, v))) <= 1e-12
        if x_before is not None and not np.array_equal(x_before, sch.x_curr):
            updates.append(t)
    assert updates == [7, 10, 13, 16]          # t_p^(i) = m + i*dt (reading Z9)
    assert sch.t_prev == 13 and sch.t_curr == 16


def test_first_window_uses_warmup_pair():
    w = syn.TINY
    L = O.make_layout(w.batch, w.heads, w.head_dim, w.prefix_tokens, w.frames, w.height, w.width, w.block)
    sch = O.OracleSchedule(L, T=20, m=12, dt=10, top_k=3)
    for t in range(1, 14):
        q, k, v = syn.family_s(w, step=t)
        sch.step(t, q, k, v, compute_attention=False)
    assert (sch.t_prev, sch.t_curr) == (11, 12)   # spacing 1 in the first window (reading Z10)
    assert sch.keep.shape == (1, 2, 4)


def test_drifting_family_s_moves_the_fitted_intensities():
    """synthetic.family_s(drift>0) gives the oracle pipeline a real trend over denoising steps:
    the pooled-statistic fits move far more across t than with noise-only steps, and drift = 0 is
    byte-identical to the plain generator."""
    import synthetic as syn
    w = syn.TINY
    L = O.make_layout(1, 2, 64, 0, 4, 8, 8, 64)
    assert all(np.array_equal(a.float().numpy(), b.float().numpy())
               for a, b in zip(syn.family_s(w, step=5), syn.family_s(w, step=5, drift=0.0)))

    def spread(drift):
        xs = []
        for t in (13, 25, 37, 49):
            q, k, _ = syn.family_s(w, step=t, drift=drift)
            xs.append(O.fit_mixture(O.pooled_block_stats(q, k, L), L))
        xs = np.stack(xs)
        return float(np.abs(xs[-1] - xs[0]).mean())
    assert spread(0.8) > 2.0 * spread(0.0)
