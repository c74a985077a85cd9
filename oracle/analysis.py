"""Oracle: analysis metrics of the paper's ablations (App. A) -- TEST INFRASTRUCTURE ONLY.

Plain fp64 numpy, written from PAPER.md; shares no code with the CUDA path.

* ``rel_frobenius``  ||A - B|| / ||B|| with the matrix 2-norm read as Frobenius (reading Z20).  It is
  the difference error ratio DER(t) = ||S^(t) - S^(12)|| / ||S^(12)|| (App. A) and the
  normalised reconstruction error NRE(t) = ||S_hat^(t) - S_GT^(t)|| / ||S_GT^(t)||.
* ``linearity_nre``  NRE = sqrt((1/N_t) sum_t (x_k^(t) - x_hat_k^(t))^2) / (max_t x_k^(t) - min_t x_k^(t))
  (App. A) with x_hat the Eq. 6/7 linear prediction from the
  window's two anchors (reading Z28: the "linear prediction" of P:886 is the method's own).
"""
from __future__ import annotations

import numpy as np

from .layout import Layout


def rel_frobenius(A: np.ndarray, B: np.ndarray) -> float:
    """||A - B||_F / ||B||_F in fp64; 0 if both differences and B vanish, +inf if only B vanishes."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    d = np.sqrt(np.sum((A - B) ** 2))
    b = np.sqrt(np.sum(B ** 2))
    if b == 0.0:
        return 0.0 if d == 0.0 else float("inf")
    return float(d / b)


def der(S_t: np.ndarray, S_ref: np.ndarray) -> float:
    """Difference error ratio (App. A): deviation of the map at step t from the warm-up map."""
    return rel_frobenius(S_t, S_ref)


def reconstruction_nre(S_hat: np.ndarray, S_gt: np.ndarray) -> float:
    """Normalised reconstruction error of Eq. 5's map (App. A)."""
    return rel_frobenius(S_hat, S_gt)


def linearity_nre(x_prev: np.ndarray, x_curr: np.ndarray, t_prev: int, t_curr: int, x_traj: np.ndarray,
                  t_steps, L: Layout) -> np.ndarray:
    """Per C/D pattern k (3n-1 of them; frame intensities are not predicted):
    x_hat^(t) = x_c + (x_c - x_p)/(t_c - t_p) * (t - t_c)   (Eq. 6)
    NRE_k = sqrt(mean_s (x^(t_s) - x_hat^(t_s))^2) / (max_s x^(t_s) - min_s x^(t_s)); NaN for a flat k.
    x_prev, x_curr: [p]; x_traj: [S, p] true fits at the steps t_steps."""
    npool = 3 * L.n - 1
    xp = np.asarray(x_prev, dtype=np.float64)[:npool]
    xc = np.asarray(x_curr, dtype=np.float64)[:npool]
    X = np.asarray(x_traj, dtype=np.float64)[:, :npool]
    t = np.asarray(t_steps, dtype=np.float64)
    slope = (xc - xp) / float(t_curr - t_prev)
    Xhat = xc[None, :] + slope[None, :] * (t[:, None] - float(t_curr))
    rms = np.sqrt(np.mean((X - Xhat) ** 2, axis=0))
    rng = X.max(axis=0) - X.min(axis=0)
    out = np.full(npool, np.nan)
    ok = rng > 0
    out[ok] = rms[ok] / rng[ok]
    return out
