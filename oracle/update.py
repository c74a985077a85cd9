"""O10 -- online mask update / sparsity-map reconstruction (oracle; test infrastructure only).

Eq. 5 (§5.1): A_hat^(t_p^(i+1))(p,q) = A_masked(p,q) where M(p,q) = 0, else
A_hat^(t_p^(i))(p,q); seed A_hat^(t_p^(0)) = A^(m).  Readings Z11, Z12: A_masked is
normalised over the unmasked entries only; with the POOLED statistic the block-level analog
is exact because M is block-constant: the fresh map W is row-renormalised over the selected
blocks of row i (sequential fp64 sum in ascending j), and
  S_hist[i,j] <- sel(i,j) ? W[i,j] / sum_{j' sel} W[i,j'] : S_hist[i,j].
Then X^(t_p) = fit(S_hist) (Alg. 1) and the intensity pair rolls:
  x_prev <- x_curr, x_curr <- X^(t_p)  (reading Z9/Z10).
"""
from __future__ import annotations

import numpy as np

from .fit import fit_mixture
from .layout import Layout


def reconstruct_history(W_fresh, hist, masks, masked_renorm: bool = True):
    """Eq. 5 at block level for every head: returns the new history [.., n, n] (fp64)."""
    W = np.asarray(W_fresh, dtype=np.float64)
    Hh = np.array(hist, dtype=np.float64, copy=True)
    masks = np.asarray(masks, dtype=bool)
    lead = W.shape[:-2]
    n = W.shape[-1]
    Wf, Hf, Mf = W.reshape(-1, n, n), Hh.reshape(-1, n, n), masks.reshape(-1, n, n)
    for t in range(Wf.shape[0]):
        for i in range(n):
            js = np.nonzero(Mf[t, i])[0]
            if len(js) == 0:
                continue
            if masked_renorm:
                acc = 0.0
                for j in js:
                    acc = acc + Wf[t, i, j]
                for j in js:
                    Hf[t, i, j] = Wf[t, i, j] / acc if acc > 0 else 0.0
            else:
                Hf[t, i, js] = Wf[t, i, js]
    return Hf.reshape(lead + (n, n))


def update_online_mask(W_fresh, hist, masks, x_prev, x_curr, L: Layout, lam: float = 1e-8,
                       masked_renorm: bool = True):
    """Returns (new_hist, new_x_prev, new_x_curr)."""
    new_hist = reconstruct_history(W_fresh, hist, masks, masked_renorm)
    X = fit_mixture(new_hist, L, lam)
    return new_hist, np.array(x_curr, dtype=np.float64, copy=True), X
