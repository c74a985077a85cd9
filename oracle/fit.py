"""O3 / O4 -- pattern bases, design matrix, normal equations, solve (oracle; test infra only).

Bases (§4.2, App. B), 0-based indices (reading Z4):
  C_k, k = 0..2n-2:  C_k(i,j) = 1 iff j - i = delta_k,  delta_k = k - (n-1)
  D_k, k = 0..n-1:   D_k(i,j) = 1 iff j = k
  E_r, r = 0..F-1:   E_r(i,j) = 1 iff (i,j) in [a_r,b_r]^2       (reading Z5 for [a_r,b_r])
Design matrix M = [vec C_k, vec D_k, vec E_r], vec = row-major (i*n + j).
Objective (Eq. 4; App. B): X = argmin ||vec U - M X||^2, Tikhonov
  M^T M <- M^T M + lambda I, lambda = 1e-8 (App. B).
Normal equations M^T M X = M^T vec U.
Closed-form Gram blocks (App. B; the C^T E, D^T E and overlapping E^T E entries
are not printed in the paper and are derived by counting support intersections -- pinned by
exact equality with the materialized M^T M in tests):
  [C^T C]_kk = n - |delta_k|; [D^T D] = n I; [C^T D]_kj = 1 iff 0 <= j - delta_k <= n-1;
  [C^T E]_kr = max(0, L_r - |delta_k|); [D^T E]_jr = L_r iff a_r <= j <= b_r;
  [E^T E]_rr' = |[a_r,b_r] cap [a_r',b_r']|^2;  L_r = b_r - a_r + 1.
RHS: diagonal sums over D_k, column sums, square sums.
Solver chain (App. B): Cholesky -> LU with partial pivoting -> SVD pseudo-inverse.
NAE (§4.2, reading Z20 Frobenius): ||U - M X||_F / ||U||_F.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .layout import Layout


def basis_C(n: int, k: int) -> np.ndarray:
    d = k - (n - 1)
    C = np.zeros((n, n))
    for i in range(n):
        j = i + d
        if 0 <= j < n:
            C[i, j] = 1.0
    return C


def basis_D(n: int, k: int) -> np.ndarray:
    Dm = np.zeros((n, n))
    Dm[:, k] = 1.0
    return Dm


def basis_E(L: Layout, r: int) -> np.ndarray:
    n = L.n
    a, b = L.frame_blocks(r)
    E = np.zeros((n, n))
    E[a:b + 1, a:b + 1] = 1.0
    return E


def design_matrix(L: Layout) -> np.ndarray:
    """Materialized M (n^2 x p).  Oracle-scale only."""
    n = L.n
    cols = [basis_C(n, k).ravel() for k in range(2 * n - 1)]
    cols += [basis_D(n, k).ravel() for k in range(n)]
    cols += [basis_E(L, r).ravel() for r in range(L.frames)]
    return np.stack(cols, axis=1)


def gram_materialized(L: Layout, lam: float = 0.0) -> np.ndarray:
    M = design_matrix(L)
    return M.T @ M + lam * np.eye(M.shape[1])


def gram_closed_form(L: Layout, lam: float = 1e-8) -> np.ndarray:
    """M^T M + lambda I without materializing M (App. B)."""
    n, F = L.n, L.frames
    p = 3 * n - 1 + F
    G = np.zeros((p, p))
    oC, oD, oE = 0, 2 * n - 1, 3 * n - 1
    fr = [L.frame_blocks(r) for r in range(F)]
    for k in range(2 * n - 1):
        d = k - (n - 1)
        G[oC + k, oC + k] = n - abs(d)                           # C^T C
        for j in range(n):                                        # C^T D
            if 0 <= j - d <= n - 1:
                G[oC + k, oD + j] = G[oD + j, oC + k] = 1.0
        for r, (a, b) in enumerate(fr):                           # C^T E (derived, counted)
            G[oC + k, oE + r] = G[oE + r, oC + k] = max(0, (b - a + 1) - abs(d))
    for j in range(n):
        G[oD + j, oD + j] = n                                     # D^T D
        for r, (a, b) in enumerate(fr):                           # D^T E (derived, counted)
            if a <= j <= b:
                G[oD + j, oE + r] = G[oE + r, oD + j] = b - a + 1
    for r, (a, b) in enumerate(fr):                               # E^T E (P:1165-1169 + overlap)
        for r2, (a2, b2) in enumerate(fr):
            ov = max(0, min(b, b2) - max(a, a2) + 1)
            G[oE + r, oE + r2] = ov * ov
    return G + lam * np.eye(p)


def rhs(U: np.ndarray, L: Layout) -> np.ndarray:
    """M^T vec U by partitioned sums for one n x n map."""
    U = np.asarray(U, dtype=np.float64)
    n = L.n
    r_c = np.array([np.trace(U, offset=k - (n - 1)) for k in range(2 * n - 1)])   # sum over D_k
    r_d = U.sum(axis=0)                                                          # column sums
    r_e = []
    for r in range(L.frames):
        a, b = L.frame_blocks(r)
        r_e.append(U[a:b + 1, a:b + 1].sum())                                    # square sums
    return np.concatenate([r_c, r_d, np.array(r_e)])


def rhs_materialized(U: np.ndarray, L: Layout) -> np.ndarray:
    return design_matrix(L).T @ np.asarray(U, dtype=np.float64).ravel()


def solve_normal(G: np.ndarray, r: np.ndarray) -> tuple[np.ndarray, str]:
    """Adaptive solve of G X = r (App. B): Cholesky, else LU, else pinv."""
    try:
        c = sla.cho_factor(G, lower=True, check_finite=True)
        x = sla.cho_solve(c, r)
        if np.all(np.isfinite(x)):
            return x, "cholesky"
    except (np.linalg.LinAlgError, ValueError):
        pass
    try:
        lu = sla.lu_factor(G, check_finite=True)
        x = sla.lu_solve(lu, r)
        if np.all(np.isfinite(x)):
            return x, "lu"
    except (np.linalg.LinAlgError, ValueError):
        pass
    x = np.linalg.pinv(G, rcond=max(G.shape) * np.finfo(float).eps) @ r
    return x, "pinv"


def fit_mixture(U, L: Layout, lam: float = 1e-8, materialize: bool | None = None):
    """X [B,H,p] = (M^T M + lambda I)^-1 M^T vec U for every head (Eq. 4; Alg. 1)."""
    U = np.asarray(U, dtype=np.float64)
    if materialize is None:
        materialize = L.n <= 48
    if materialize:
        M = design_matrix(L)
        G = M.T @ M + lam * np.eye(M.shape[1])
    else:
        G = gram_closed_form(L, lam)
    lead = U.shape[:-2]
    Uf = U.reshape((-1,) + U.shape[-2:])
    X = np.empty((Uf.shape[0], G.shape[0]))
    for t in range(Uf.shape[0]):
        r = (M.T @ Uf[t].ravel()) if materialize else rhs(Uf[t], L)
        X[t], _ = solve_normal(G, r)
    return X.reshape(lead + (G.shape[0],))


def reconstruct_from_x(x: np.ndarray, L: Layout) -> np.ndarray:
    """M X reshaped to n x n (the mixture of Eq. 3 without R)."""
    n = L.n
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros((n, n))
    for k in range(2 * n - 1):
        out += x[k] * basis_C(n, k)
    for k in range(n):
        out += x[2 * n - 1 + k] * basis_D(n, k)
    for r in range(L.frames):
        out += x[3 * n - 1 + r] * basis_E(L, r)
    return out


def nae(U: np.ndarray, x: np.ndarray, L: Layout) -> float:
    """NAE = ||R||_F / ||U||_F with R = U - sum(c C + d D + e E) (§4.2)."""
    U = np.asarray(U, dtype=np.float64)
    R = U - reconstruct_from_x(x, L)
    return float(np.linalg.norm(R) / np.linalg.norm(U))
