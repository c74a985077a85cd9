"""O5-O10 assembled: Algorithm 1 for one layer, in fp64 (oracle; test infra only).

Same schedule semantics as DESIGN.md / SURVEY 8(c): warm-up t <= m full attention, statistics and
fits at t = m-1 and m, keep decision at m, prediction for t > m from (x_prev, x_curr),
reconstruction + refit at t_p^(i) = m + i*dt, i >= 1 (readings Z9-Z12).
"""
from __future__ import annotations

import numpy as np

from .attention import masked_attention
from .fit import fit_mixture
from .layout import Layout
from .predict import SELECT_TOPK, keep_frames, predict_block_mask
from .stats import exact_sparsity_masked, pooled_block_stats
from .update import reconstruct_history


class OracleSchedule:
    def __init__(self, L: Layout, T=50, m=12, dt=10, top_k=1, mode=SELECT_TOPK, param=0.0, tau_e=0.0,
                 lam=1e-8, diag_guard=True, masked_renorm=True, stat="pooled", eta=1e-4):
        self.L, self.T, self.m, self.dt = L, T, m, dt
        self.top_k, self.mode, self.param, self.tau_e, self.lam = top_k, mode, param, tau_e, lam
        self.guard, self.renorm = diag_guard, masked_renorm
        self.stat, self.eta = stat, eta
        self.x_prev = self.x_curr = self.keep = self.hist = None
        self.t_prev = self.t_curr = -1

    def mask_for(self, t):
        L = self.L
        if t <= self.m:
            return np.ones((L.batch, L.heads, L.n, L.n), dtype=bool)
        return predict_block_mask(self.x_prev, self.x_curr, self.t_prev, self.t_curr, t, self.keep, L,
                                  self.mode, self.top_k, self.param, self.guard)

    def _stat(self, q, k, mask):
        if self.stat == "pooled":
            return pooled_block_stats(q, k, self.L)
        S, _ = exact_sparsity_masked(q, k, mask, self.L, self.eta)     # Eq. 2 on (masked) P; NaN off-mask
        return -S                                                      # reading Z3

    def step(self, t, q, k, v, mask_override=None, compute_attention=True):
        L = self.L
        mask = self.mask_for(t) if mask_override is None else mask_override
        out = masked_attention(q, k, v, mask, L) if compute_attention else (None, None)
        if t == self.m - 1:
            self.x_prev, self.t_prev = fit_mixture(self._stat(q, k, mask), L, self.lam), t
        elif t == self.m:
            W = self._stat(q, k, mask)
            self.x_curr, self.t_curr = fit_mixture(W, L, self.lam), t
            self.keep = keep_frames(self.x_prev, self.x_curr, L, self.tau_e)
            self.hist = W
        elif t > self.m and (t - self.m) % self.dt == 0:
            W = self._stat(q, k, mask)
            self.hist = reconstruct_history(W, self.hist, mask, self.renorm)
            self.x_prev, self.x_curr = self.x_curr, fit_mixture(self.hist, L, self.lam)
            self.t_prev, self.t_curr = self.t_curr, t
        return mask, out
