"""Algorithm 1 of MOD-DiT for one attention layer, driving the C-ABI kernels.

    t = 1..m           full attention: K4 on all-ones index lists (FlashAttention-2 in the paper)
    t = m-1, m         pooled statistics + mixture fit  X^(m-1), X^(m)
    t = m              block-diagonal keep decision; history seeded with W^(m)
    t > m              mask = predict(x_prev, x_curr; t) (Eq. 6/7 + §5.3) -> block-sparse attention
    t = t_p^(i) = m + i*dt (i >= 1)   after the attention: fresh statistics, Eq. 5 merge, refit, roll
                                      (reading Z9: t_p^(i) = m + i*dt, not "t mod dt == 0"; Z11: the
                                      attention at t_p uses the previous window's prediction)
All state is plain device tensors (checkpointable with torch.save); everything is stream-ordered and
no host synchronisation happens inside ``step``.
"""
from __future__ import annotations

import dataclasses

import torch

from .plan import Plan


@dataclasses.dataclass
class ScheduleState:
    t_prev: int = -1
    t_curr: int = -1
    x_prev: torch.Tensor | None = None
    x_curr: torch.Tensor | None = None
    keep: torch.Tensor | None = None
    hist: torch.Tensor | None = None
    W_warm: torch.Tensor | None = None


class Schedule:
    def __init__(self, plan: Plan, T: int = 50, m: int = 12, dt: int = 10, top_k: int | None = None,
                 select_mode: int | None = None, select_param: float | None = None, stat: str = "pooled",
                 eta: float = 1e-4, precision: str = "bf16", overlap_k1: bool = True):
        if not (1 <= m < T) or dt < 1 or m < 2:
            raise ValueError(f"bad schedule T={T} m={m} dt={dt}")
        if stat not in ("pooled", "exact"):
            raise ValueError(f"stat={stat!r} must be 'pooled' or 'exact'")
        if precision not in ("bf16", "q8"):
            raise ValueError(f"precision={precision!r} must be 'bf16' or 'q8'")
        if precision == "q8" and stat == "exact":
            raise ValueError("precision='q8' needs stat='pooled' (the exact statistic thresholds the bf16 lse)")
        if stat == "exact" and plan.config["masked_renorm"]:
            raise ValueError("stat='exact' needs a Plan with masked_renorm=False: the masked map is already "
                             "renormalised by the sparse attention's lse (reading Z12)")
        self.P, self.T, self.m, self.dt = plan, T, m, dt
        self.stat, self.eta, self.precision = stat, eta, precision
        self.overlap_k1 = overlap_k1   # K1 on a side stream beside K4 at update steps (pooled statistic)
        self._qbuf = None
        self.sel = dict(top_k=top_k, select_mode=select_mode, select_param=select_param)
        self.state = ScheduleState()
        self._dense = None
        self.last_mask = None

    def is_update_step(self, t: int) -> bool:
        """t is a prediction step t_p^(i) = m + i*dt with i >= 1."""
        return t > self.m and (t - self.m) % self.dt == 0

    def dense_mask(self):
        if self._dense is None:
            self._dense = self.P.dense_mask()
        return self._dense

    def step(self, t: int, q, k, v, out=None, lse=None):
        """One denoising step of one attention layer; returns (O, lse)."""
        P, S = self.P, self.state
        if not 1 <= t <= self.T:
            raise ValueError(f"t={t} outside [1, {self.T}]")
        if t <= self.m:
            rp, ci = self.dense_mask()
            o, l = P.block_sparse_attn_fwd(q, k, v, rp, ci, out=out, lse=lse)   # K4 on the all-ones list
            if t == self.m - 1:
                S.W_warm = self._stat(q, k, l, rp, ci)
                S.x_prev, S.t_prev = P.fit_mixture(S.W_warm), t
            elif t == self.m:
                W = self._stat(q, k, l, rp, ci)
                S.x_curr, S.t_curr = P.fit_mixture(W), t
                S.keep = P.keep_frames(S.x_prev, S.x_curr)
                S.hist = W                                    # A_hat^(t_p^(0)) = A^(m)
                S.W_warm = None
            self.last_mask = (rp, ci)
            return o, l
        rp, ci = P.predict_block_mask(S.x_prev, S.x_curr, S.t_prev, S.t_curr, t, S.keep, **self.sel)
        W_side = None
        if self.is_update_step(t) and self.stat == "pooled" and self.overlap_k1:
            # K1 reads only this step's Q, K: it runs on a side stream beside K4 (its HBM-bound pool pass fills
            # the SMs' spare issue and bandwidth next to the compute-bound attention); K3 joins both
            W_side = self._pooled_side(q, k)
        if self.precision == "q8":   # sparse steps on the Sage-style quantized path (reading Z30)
            if self._qbuf is None:
                self._qbuf = P.quant_buffer()
            P.quantize_qkv(q, k, v, out=self._qbuf)
            o, l = P.block_sparse_attn_fwd_q8(self._qbuf, rp, ci, out=out, lse=lse)
        else:
            o, l = P.block_sparse_attn_fwd(q, k, v, rp, ci, out=out, lse=lse)
        if self.is_update_step(t):
            if W_side is not None:
                torch.cuda.current_stream().wait_stream(self._side)
                W = W_side
            else:
                W = self._stat(q, k, l, rp, ci)
            P.update_online_mask(W, rp, ci, S.hist, S.x_prev, S.x_curr)
            S.t_prev, S.t_curr = S.t_curr, t
        self.last_mask = (rp, ci)
        return o, l

    def _pooled_side(self, q, k):
        """K1 (pooled statistic) enqueued on the driver's side stream after everything already on the current
        stream (so the previous step's reads of its output are complete); the caller joins before K3."""
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        self._side.wait_stream(main)
        with torch.cuda.stream(self._side):
            W = self.P.collect_block_stats(q, k)
        W.record_stream(main)
        return W

    def _stat(self, q, k, lse, rp, ci):
        """Block statistic U of this step: POOLED (north_star (1)) or EXACT Eq. 2 from the attention's lse
        over the listed blocks (dense list at warm-up, sparse list at t_p: Eq. 5's A_masked)."""
        if self.stat == "pooled":
            return self.P.collect_block_stats(q, k)
        return self.P.collect_exact_sparsity(q, k, lse, rp, ci, self.eta)

    def state_dict(self) -> dict:
        return {f.name: getattr(self.state, f.name) for f in dataclasses.fields(self.state) if f.name != "W_warm"}

    def load_state_dict(self, d: dict):
        for k, v in d.items():
            setattr(self.state, k, v)
