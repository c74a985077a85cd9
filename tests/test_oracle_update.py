"""Pins for oracle O10 (Eq. 5 reconstruction + refit) -- no GPU.  SPEC.md S:398-424."""
import numpy as np

import oracle as O


def _maps(n=4, seed=0):
    rng = np.random.default_rng(seed)
    W = rng.random((1, 1, n, n))
    W /= W.sum(-1, keepdims=True)
    Hh = rng.random((1, 1, n, n))
    return W, Hh


def test_all_pass_gives_fresh_map():
    W, Hh = _maps()
    m = np.ones_like(W, dtype=bool)
    assert np.allclose(O.reconstruct_history(W, Hh, m), W, atol=1e-15)
    assert np.array_equal(O.reconstruct_history(W, Hh, m, masked_renorm=False), W)


def test_all_block_keeps_history():
    W, Hh = _maps()
    m = np.zeros_like(W, dtype=bool)
    assert np.array_equal(O.reconstruct_history(W, Hh, m), Hh)


def test_two_by_two_selection_no_blending():
    W, Hh = _maps(2)
    m = np.zeros((1, 1, 2, 2), dtype=bool)
    m[0, 0, 0, 0] = True
    out = O.reconstruct_history(W, Hh, m, masked_renorm=False)
    assert out[0, 0, 0, 0] == W[0, 0, 0, 0]
    assert out[0, 0, 0, 1] == Hh[0, 0, 0, 1] and out[0, 0, 1, 0] == Hh[0, 0, 1, 0] and out[0, 0, 1, 1] == Hh[0, 0, 1, 1]
    # masked renormalisation: a single selected block in a row carries the whole row mass
    out = O.reconstruct_history(W, Hh, m)
    assert out[0, 0, 0, 0] == 1.0


def test_renormalised_rows_sum_to_one_over_selection_and_idempotent():
    W, Hh = _maps(6, 1)
    rng = np.random.default_rng(2)
    m = rng.random(W.shape) < 0.4
    m |= np.eye(6, dtype=bool)
    out = O.reconstruct_history(W, Hh, m)
    assert np.allclose(np.where(m, out, 0).sum(-1), 1.0, atol=1e-14)
    assert np.array_equal(out[~m], Hh[~m])
    assert np.array_equal(O.reconstruct_history(W, out, m), out)


def test_update_rolls_intensities():
    L = O.make_layout(1, 1, 8, 0, 2, 1, 8, 4)
    W, Hh = _maps(L.n, 3)
    m = np.ones_like(W, dtype=bool)
    xp, xc = np.zeros((1, 1, L.p)), np.ones((1, 1, L.p))
    h2, xp2, xc2 = O.update_online_mask(W, Hh, m, xp, xc, L)
    assert np.array_equal(xp2, xc)
    assert np.allclose(xc2, O.fit_mixture(h2, L))
