"""Host-resident activations through the hot path, overlapped by head chunks (serving form of one step).

Every step of MOD-DiT's hot path is per (batch, head) (K1-K4 and the fit have no
cross-head reduction), so a step over host-resident Q, K, V can be cut into head chunks and run as a
three-stage pipeline on three CUDA streams:

    h2d stream      Q, K, V of chunk c   host (pinned) -> device
    compute stream  the caller's step on chunk c (``Plan`` calls on head-slice views)
    d2h stream      O of chunk c         device -> host (pinned)

Chunk c+1's upload runs while chunk c computes and chunk c-1 downloads, so a step costs about
max(PCIe upload, compute, download) instead of their sum.  Events order the reuse of the device
buffers across consecutive ``run`` calls (the upload of step s+1 into chunk c waits for step s's compute
on chunk c; step s+1's compute on chunk c waits for step s's download of chunk c).  This module only
orders copies and launches: all arithmetic is in libmoddit.so behind ``Plan``.
"""
from __future__ import annotations

import dataclasses

import torch

from .plan import LayoutSpec, Plan


class HeadChunkPipeline:
    """Pipelined host -> device -> host execution of a per-head step over ``chunks`` head chunks.

    ``layout`` is the full problem (B must be 1 so that a head range is one contiguous slab of every
    [B, H, ...] tensor); ``plan_kw`` configure the per-chunk ``Plan`` (one plan of H/chunks heads,
    reused for every chunk).  ``q, k, v, o`` are the device tensors the step reads and writes.
    """

    def __init__(self, layout, chunks: int, **plan_kw):
        spec = LayoutSpec.from_any(layout)
        if spec.batch != 1:
            raise ValueError("HeadChunkPipeline needs batch 1 (head slices must be contiguous)")
        if spec.heads % chunks:
            raise ValueError(f"heads={spec.heads} not divisible by chunks={chunks}")
        self.spec, self.chunks, self.hc = spec, chunks, spec.heads // chunks
        self.plan = Plan(dataclasses.replace(spec, heads=self.hc), **plan_kw)
        dev = torch.device(f"cuda:{self.plan.device}")
        shape = (1, spec.heads, spec.tokens, spec.head_dim)
        self.q, self.k, self.v, self.o = (torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(4))
        self.s_h2d, self.s_comp, self.s_d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
        self._computed = [None] * chunks     # compute of chunk c done (its Q/K/V may be overwritten)
        self._drained = [None] * chunks      # download of chunk c done (its O may be overwritten)

    def heads(self, c: int) -> slice:
        return slice(c * self.hc, (c + 1) * self.hc)

    def run(self, hq, hk, hv, ho, step_fn):
        """One pipelined step.  ``hq, hk, hv, ho`` are pinned host tensors of the full shape;
        ``step_fn(plan, c, q_c, k_c, v_c, o_c)`` enqueues the chunk's work on the current stream.
        Returns after enqueueing; the caller's current stream is made to wait for the last download."""
        caller = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(caller)
        for c in range(self.chunks):
            hs = self.heads(c)
            with torch.cuda.stream(self.s_h2d):
                self.s_h2d.wait_event(start)
                if self._computed[c] is not None:
                    self.s_h2d.wait_event(self._computed[c])
                for dst, src in ((self.q, hq), (self.k, hk), (self.v, hv)):
                    dst[:, hs].copy_(src[:, hs], non_blocking=True)
                up = torch.cuda.Event()
                up.record(self.s_h2d)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(up)
                if self._drained[c] is not None:
                    self.s_comp.wait_event(self._drained[c])
                step_fn(self.plan, c, self.q[:, hs], self.k[:, hs], self.v[:, hs], self.o[:, hs])
                done = torch.cuda.Event()
                done.record(self.s_comp)
                self._computed[c] = done
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(done)
                ho[:, hs].copy_(self.o[:, hs], non_blocking=True)
                dr = torch.cuda.Event()
                dr.record(self.s_d2h)
                self._drained[c] = dr
        for c in range(self.chunks):
            caller.wait_event(self._drained[c])
