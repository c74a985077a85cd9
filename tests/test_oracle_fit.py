"""Pins for oracle O3/O4 (bases, design matrix, Gram, RHS, solve, NAE) -- no GPU.

Each pin is fixed by something other than the oracle itself: the paper's closed forms
(App. B), exact integer arithmetic of the materialized design matrix, exact
rational solves, SVD minimum-norm solutions and SPEC.md worked examples.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O


def lay(N_blocks_tokens=None, *, block, frames, hw, prefix=0, h=1, w=None):
    # frames x hw video tokens (+prefix); height=1, width=hw
    return O.make_layout(1, 1, 64, prefix, frames, 1, hw, block)


# ---------- bases: closed-form index sets (reading Z4)
def test_basis_supports_spec_examples():
    n = 4
    C = O.basis_C(n, 3)                         # 0-based k=3 -> delta 0: main diagonal
    assert set(zip(*np.nonzero(C))) == {(0, 0), (1, 1), (2, 2), (3, 3)}
    D = O.basis_D(n, 1)
    assert set(zip(*np.nonzero(D))) == {(0, 1), (1, 1), (2, 1), (3, 1)}
    L = lay(block=4, frames=2, hw=8)            # n = 4, two frames of 2 blocks
    assert L.n == 4
    E = O.basis_E(L, 1)
    assert set(zip(*np.nonzero(E))) == {(2, 2), (2, 3), (3, 2), (3, 3)}


def test_basis_index_sets_match_app_b_enumeration():
    # D_k of P:1217-1219: delta >= 0 -> {(i, i+delta): i in [0, n-1-delta]}; delta < 0 -> {(i-delta, i)}
    for n in (1, 2, 5, 9):
        for k in range(2 * n - 1):
            d = k - (n - 1)
            if d >= 0:
                ref = {(i, i + d) for i in range(0, n - d)}
            else:
                ref = {(i - d, i) for i in range(0, n + d)}
            assert set(zip(*np.nonzero(O.basis_C(n, k)))) == ref
            assert O.basis_C(n, k).sum() == n - abs(d)          # support size n - |delta|


def test_design_matrix_column_sums_spec():
    L = lay(block=4, frames=1, hw=8)            # n = 2, f = 1
    M = O.design_matrix(L)
    assert M.shape == (4, 6)
    assert list(M.sum(axis=0)) == [1, 2, 1, 2, 2, 4]
    L1 = lay(block=8, frames=1, hw=8)           # n = 1
    assert np.array_equal(O.design_matrix(L1), np.ones((1, 3)))


def test_design_matrix_rank_deficient():
    # sum_k C_k = J = sum_k D_k: never full column rank for n >= 2
    for L in (lay(block=4, frames=2, hw=8), lay(block=16, frames=8, hw=40)):
        M = O.design_matrix(L)
        assert np.linalg.matrix_rank(M) < M.shape[1]


# ---------- Gram: paper closed forms and exact equality with the materialized M^T M
def test_gram_paper_blocks_n4():
    L = lay(block=4, frames=2, hw=8)            # n = 4, f = 2, s = 2
    G = O.gram_closed_form(L, lam=0.0)
    n = 4
    assert list(np.diag(G)[: 2 * n - 1]) == [1, 2, 3, 4, 3, 2, 1]
    assert np.array_equal(G[2 * n - 1: 3 * n - 1, 2 * n - 1: 3 * n - 1], 4 * np.eye(4))
    assert np.array_equal(G[3 * n - 1:, 3 * n - 1:], np.diag([4.0, 4.0]))         # P:1165-1169 (b^2)


LAYOUTS = [
    (256, 64, 4, 64, 0),      # tiny: F = n = 4, aligned
    (320, 16, 8, 40, 0),      # overlapping non-aligned squares
    (1024, 32, 4, 256, 0),
    (900, 32, 9, 100, 0),     # ragged last block
    (226 + 6 * 45, 32, 6, 45, 226),   # CogVideoX-like prefix, squares smaller than 2 blocks
    (40 + 3 * 100, 64, 3, 100, 40),
]


@pytest.mark.parametrize("N,b,F,HW,P0", LAYOUTS)
def test_gram_closed_form_equals_materialized_exactly(N, b, F, HW, P0):
    L = O.make_layout(1, 1, 64, P0, F, 1, HW, b)
    assert L.N == N
    Gc = O.gram_closed_form(L, lam=0.0)
    Gm = O.gram_materialized(L, lam=0.0)
    assert np.array_equal(Gc, Gm)                 # integer-valued, exact


# ---------- RHS
def test_rhs_all_ones_spec():
    L = lay(block=4, frames=2, hw=8)
    r = O.rhs(np.ones((4, 4)), L)
    assert list(r) == [1, 2, 3, 4, 3, 2, 1, 4, 4, 4, 4, 4, 4]
    assert np.array_equal(O.rhs(np.zeros((4, 4)), L), np.zeros(13))


@pytest.mark.parametrize("N,b,F,HW,P0", LAYOUTS)
def test_rhs_equals_materialized(N, b, F, HW, P0):
    L = O.make_layout(1, 1, 64, P0, F, 1, HW, b)
    U = np.random.default_rng(1).random((L.n, L.n))
    assert np.allclose(O.rhs(U, L), O.rhs_materialized(U, L), rtol=0, atol=1e-12)


# ---------- solve
def _frac_solve(G, r):
    """Exact rational Gauss-Jordan (independent of LAPACK)."""
    p = len(r)
    A = [[Fraction(G[i][j]) for j in range(p)] + [Fraction(r[i])] for i in range(p)]
    for c in range(p):
        piv = next(i for i in range(c, p) if A[i][c] != 0)
        A[c], A[piv] = A[piv], A[c]
        inv = 1 / A[c][c]
        A[c] = [x * inv for x in A[c]]
        for i in range(p):
            if i != c and A[i][c] != 0:
                f = A[i][c]
                A[i] = [x - f * y for x, y in zip(A[i], A[c])]
    return np.array([float(A[i][p]) for i in range(p)])


def test_solve_matches_exact_rational_tiny():
    L = O.make_layout(1, 1, 64, 0, 4, 8, 8, 64)   # the tiny config: n = 4, p = 15, nullity 2
    lam = Fraction(1, 10 ** 8)
    U = np.random.default_rng(2).integers(0, 97, (4, 4)) / 97.0
    G = O.gram_closed_form(L, lam=0.0)
    Gq = [[Fraction(int(G[i, j])) + (lam if i == j else 0) for j in range(L.p)] for i in range(L.p)]
    rq = [Fraction(x).limit_denominator(10 ** 12) for x in O.rhs(U, L)]
    x_exact = _frac_solve(Gq, rq)
    x = O.fit_mixture(U[None, None], L)[0, 0]
    cond = np.linalg.cond(O.gram_closed_form(L))
    assert np.linalg.norm(x - x_exact) / np.linalg.norm(x_exact) <= 10 * cond * np.finfo(float).eps


def test_solve_zero_map_gives_zero():
    L = lay(block=4, frames=2, hw=8)
    assert np.array_equal(O.fit_mixture(np.zeros((1, 1, 4, 4)), L), np.zeros((1, 1, 13)))


def test_solve_exact_mixture_nae():
    L = lay(block=4, frames=2, hw=16)             # n = 8, f = 2
    n = L.n
    U = 0.3 * O.basis_C(n, n - 1) + 0.5 * O.basis_D(n, 3) + 0.2 * O.basis_E(L, 0)
    x = O.fit_mixture(U[None, None], L)[0, 0]
    assert O.nae(U, x, L) <= 1e-6


def test_nae_of_zero_x_is_one():
    L = lay(block=4, frames=2, hw=8)
    U = np.random.default_rng(3).random((4, 4))
    assert O.nae(U, np.zeros(L.p), L) == pytest.approx(1.0, abs=1e-15)


def test_solve_n1_symmetric():
    L = lay(block=8, frames=1, hw=8)              # n = 1, gram = all-ones + lambda I
    x = O.fit_mixture(np.full((1, 1, 1, 1), 0.6), L)[0, 0]
    assert np.allclose(x, x[0], rtol=1e-12)


@pytest.mark.parametrize("N,b,F,HW,P0", LAYOUTS)
def test_solve_matches_svd_min_norm(N, b, F, HW, P0):
    # lambda -> 0 limit of the Tikhonov solution is the Moore-Penrose minimum-norm solution
    # (App. B); independent route: SVD of the explicit M.
    L = O.make_layout(1, 1, 64, P0, F, 1, HW, b)
    U = np.random.default_rng(4).random((L.n, L.n))
    x = O.fit_mixture(U[None, None], L)[0, 0]
    M = O.design_matrix(L)
    x_mn = np.linalg.lstsq(M, U.ravel(), rcond=None)[0]
    cond = np.linalg.cond(O.gram_closed_form(L))
    tol = 1e-6 + 10 * cond * np.finfo(float).eps
    assert np.linalg.norm(x - x_mn) / np.linalg.norm(x_mn) <= tol


def test_min_norm_fit_of_all_ones_closed_form():
    # the min-norm fit of J is c = n/(3n-1), d = (2n-1)/(3n-1), e = 0
    L = lay(block=4, frames=2, hw=16)             # n = 8, F = 2
    n = L.n
    x = O.fit_mixture(np.ones((1, 1, n, n)), L)[0, 0]
    assert np.allclose(x[: 2 * n - 1], n / (3 * n - 1), atol=1e-6)
    assert np.allclose(x[2 * n - 1: 3 * n - 1], (2 * n - 1) / (3 * n - 1), atol=1e-6)
    assert np.allclose(x[3 * n - 1:], 0.0, atol=1e-6)


def test_residual_optimality():
    L = lay(block=4, frames=2, hw=16)
    rng = np.random.default_rng(5)
    U = rng.random((L.n, L.n))
    x = O.fit_mixture(U[None, None], L)[0, 0]
    M = O.design_matrix(L)
    lam = 1e-8
    f = lambda z: np.sum((U.ravel() - M @ z) ** 2) + lam * np.sum(z ** 2)
    f0 = f(x)
    for _ in range(100):
        dlt = rng.standard_normal(L.p)
        dlt *= 1e-3 / np.linalg.norm(dlt)
        assert f(x + dlt) >= f0 - 1e-12


def test_closed_form_fit_equals_materialized_fit():
    L = O.make_layout(1, 1, 64, 0, 9, 1, 100, 32)
    U = np.random.default_rng(6).random((1, 2, L.n, L.n))
    xa = O.fit_mixture(U, L, materialize=True)
    xb = O.fit_mixture(U, L, materialize=False)
    cond = np.linalg.cond(O.gram_closed_form(L))
    assert np.max(np.abs(xa - xb)) / np.max(np.abs(xa)) <= 10 * cond * np.finfo(float).eps
