"""Pins for the oracle's analysis metrics (App. A) -- no GPU.

Each pin is a closed form or a brute-force enumeration, not a retyping of the oracle's formula."""
import math

import numpy as np
import pytest

import oracle as O


def test_rel_frobenius_closed_forms():
    n = 6
    B = np.ones((n, n))
    A = B.copy()
    A[2, 3] += 0.75                       # one perturbed entry: ||A-B|| = 0.75, ||B|| = n
    assert O.rel_frobenius(A, B) == pytest.approx(0.75 / n, rel=1e-15)
    assert O.rel_frobenius(2.5 * B, B) == pytest.approx(1.5, rel=1e-15)         # A = cB -> |c - 1|
    assert O.rel_frobenius(B, B) == 0.0
    # Pythagoras: identity vs identity + all off-diagonal ones -> sqrt(n^2 - n) / sqrt(n)
    I = np.eye(n)
    assert O.rel_frobenius(np.ones((n, n)), I) == pytest.approx(math.sqrt(n - 1), rel=1e-14)
    # degenerate reference map
    Z = np.zeros((n, n))
    assert O.rel_frobenius(Z, Z) == 0.0 and O.rel_frobenius(B, Z) == math.inf


def test_rel_frobenius_brute_force_and_scale_invariance():
    rng = np.random.default_rng(5)
    A, B = rng.random((5, 7)), rng.random((5, 7))
    num = den = 0.0
    for i in range(5):                     # plain loops over entries
        for j in range(7):
            num += (A[i, j] - B[i, j]) ** 2
            den += B[i, j] ** 2
    assert O.rel_frobenius(A, B) == pytest.approx(math.sqrt(num) / math.sqrt(den), rel=1e-14)
    assert O.rel_frobenius(3 * A, 3 * B) == pytest.approx(O.rel_frobenius(A, B), rel=1e-14)


def test_der_of_a_linear_drift_is_linear_in_t():
    """S^(t) = S^(12) + (t - 12) D  =>  DER(t) = (t - 12) ||D|| / ||S^(12)||."""
    rng = np.random.default_rng(1)
    S12 = rng.random((8, 8))
    D = rng.standard_normal((8, 8)) * 1e-2
    r = np.linalg.norm(D) / np.linalg.norm(S12)
    for t in (12, 13, 20, 50):
        assert O.der(S12 + (t - 12) * D, S12) == pytest.approx((t - 12) * r, rel=1e-12, abs=1e-15)


def test_reconstruction_nre_counts_only_unselected_blocks():
    """Eq. 5 without renormalisation keeps history outside the mask: the reconstruction error is the
    history's deviation on the unselected blocks (brute force), 0 when every block is selected."""
    rng = np.random.default_rng(2)
    n = 5
    GT, Hh = rng.random((1, 1, n, n)), rng.random((1, 1, n, n))
    sel = rng.random((1, 1, n, n)) < 0.4
    S_hat = O.reconstruct_history(GT, Hh, sel, masked_renorm=False)
    num = sum((Hh[0, 0, i, j] - GT[0, 0, i, j]) ** 2 for i in range(n) for j in range(n) if not sel[0, 0, i, j])
    den = sum(GT[0, 0, i, j] ** 2 for i in range(n) for j in range(n))
    assert O.reconstruction_nre(S_hat, GT) == pytest.approx(math.sqrt(num / den), rel=1e-14)
    all_sel = np.ones_like(sel)
    assert O.reconstruction_nre(O.reconstruct_history(GT, Hh, all_sel, masked_renorm=False), GT) == 0.0


def _layout():
    return O.make_layout(1, 1, 64, 0, 4, 8, 8, 64)        # tiny: n = 4, p = 15


def test_linearity_nre_zero_on_lines_and_nan_when_flat():
    L = _layout()
    npool = 3 * L.n - 1
    alpha, beta = np.linspace(-1, 1, L.p), np.linspace(0.5, -2, L.p)
    beta[0] = 0.0                                           # pattern 0 is flat -> NaN (range 0)
    line = lambda t: alpha + beta * t                       # noqa: E731
    ts = list(range(23, 33))
    traj = np.stack([line(t) for t in ts])
    out = O.linearity_nre(line(12), line(22), 12, 22, traj, ts, L)
    assert out.shape == (npool,)
    assert math.isnan(out[0])
    assert np.all(np.abs(out[1:]) < 1e-12)


def test_linearity_nre_secant_of_a_quadratic():
    """x(t) = t^2, anchors 12 and 22: the secant's residual is (t - 12)(t - 22) (closed form), so the
    NRE over 23..32 is sqrt(mean((t-12)^2 (t-22)^2)) / (32^2 - 23^2)."""
    L = _layout()
    ts = np.arange(23, 33)
    traj = np.stack([np.full(L.p, float(t * t)) for t in ts])
    out = O.linearity_nre(np.full(L.p, 144.0), np.full(L.p, 484.0), 12, 22, traj, ts, L)
    want = math.sqrt(np.mean([((t - 12) * (t - 22)) ** 2 for t in ts])) / (32 ** 2 - 23 ** 2)
    assert np.allclose(out, want, rtol=1e-13)


def test_linearity_nre_is_affine_invariant():
    L = _layout()
    rng = np.random.default_rng(3)
    xp, xc = rng.standard_normal(L.p), rng.standard_normal(L.p)
    ts = [13, 14, 17, 21]
    traj = rng.standard_normal((4, L.p))
    a, b = -3.5, 7.0
    o1 = O.linearity_nre(xp, xc, 11, 12, traj, ts, L)
    o2 = O.linearity_nre(a * xp + b, a * xc + b, 11, 12, a * traj + b, ts, L)
    assert np.allclose(o1, o2, rtol=1e-12)
