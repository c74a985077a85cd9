"""Multi-GPU plumbing of the hot path: head partitioning and the Ulysses all-to-all.

Every step of MOD-DiT is per (batch, head) -- statistics, fit, prediction, update and attention
(§4.1 P:202 "We process each attention head independently"; §5.3 P:439-442 the layer mask
is the concatenation of per-head masks).  The path therefore shards by heads with no collective
on the data path.  A collective appears only when the activations arrive sequence-sharded (the
usual DiT sequence parallelism): then a Ulysses all-to-all turns [B, N/P, H, D] sequence shards
into [B, H/P, N, D] head shards before the hot path and back afterwards.  The all-to-all runs on
NCCL through torch.distributed (NVLink 5 / NVSwitch on a B200 node); the pack / unpack relayouts
around it are libmoddit kernels (csrc/ulysses.cu).  The CPU gloo tests swap in a torch relayout.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_range(heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous head block [h0, h1) owned by ``rank`` (heads must divide evenly)."""
    if heads % world:
        raise ValueError(f"heads={heads} not divisible by world size {world}")
    per = heads // world
    return rank * per, (rank + 1) * per


def lpt_head_assignment(cost, world: int) -> list[list[int]]:
    """Greedy longest-processing-time assignment of heads to ranks by per-head cost (e.g. mask nnz).
    Returns, per rank, the sorted list of heads it owns.  Deterministic (ties by head index)."""
    order = sorted(range(len(cost)), key=lambda h: (-float(cost[h]), h))
    loads = [0.0] * world
    out = [[] for _ in range(world)]
    for h in order:
        r = min(range(world), key=lambda i: (loads[i], i))
        loads[r] += float(cost[h])
        out[r].append(h)
    return [sorted(x) for x in out]


def _world(group) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


class KernelRelayout:
    """The pack / unpack around the all-to-all, run by libmoddit's relayout kernels (include/moddit.h
    ``mod_ulysses_*``).  Inputs are contiguous bf16 CUDA tensors; each call allocates its output."""

    @staticmethod
    def _run(fn, src, shape, *dims, out=None):
        from ._lib import check, lib
        import ctypes as C
        if not (src.is_cuda and src.dtype == torch.bfloat16 and src.is_contiguous()):
            raise ValueError(f"Ulysses relayout needs a contiguous bf16 CUDA tensor, got {src.dtype} {src.device}")
        if out is not None and (tuple(out.shape) != tuple(shape) or out.dtype != src.dtype or not out.is_contiguous()):
            raise ValueError(f"out must be a contiguous bf16 tensor of shape {tuple(shape)}")
        dst = torch.empty(shape, dtype=src.dtype, device=src.device) if out is None else out
        check(getattr(lib, fn)(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), *dims,
                               C.c_void_p(torch.cuda.current_stream(src.device).cuda_stream)))
        return dst

    def seq_pack(self, x_seq, P):                 # [B,Ns,H,D] -> [P,B,Ns,H/P,D]
        B, Ns, H, D = x_seq.shape
        return self._run("mod_ulysses_seq_pack", x_seq, (P, B, Ns, H // P, D), B, Ns, H, D, P)

    def seq_unpack(self, recv, out=None):         # [P,B,Ns,Hp,D] -> [B,Hp,P*Ns,D]
        P, B, Ns, Hp, D = recv.shape
        return self._run("mod_ulysses_seq_unpack", recv, (B, Hp, P * Ns, D), B, Ns, Hp, D, P, out=out)

    def head_pack(self, x_head, P, out=None):     # [B,Hp,N,D] -> [P,B,N/P,Hp,D]
        B, Hp, N, D = x_head.shape
        return self._run("mod_ulysses_head_pack", x_head, (P, B, N // P, Hp, D), B, N, Hp, D, P, out=out)

    def head_unpack(self, recv, out=None):        # [P,B,Ns,Hp,D] -> [B,Ns,P*Hp,D]
        P, B, Ns, Hp, D = recv.shape
        return self._run("mod_ulysses_head_unpack", recv, (B, Ns, P * Hp, D), B, Ns, Hp, D, P, out=out)

    def seq_pack_heads(self, x_seq, h0, Hc, P, out=None):   # heads [h0, h0+Hc) of [B,Ns,H,D] -> [P,B,Ns,Hc/P,D]
        B, Ns, H, D = x_seq.shape
        return self._run("mod_ulysses_seq_pack_heads", x_seq, (P, B, Ns, Hc // P, D), B, Ns, H, h0, Hc, D, P, out=out)

    def head_unpack_heads(self, recv, x_seq, h0):        # [P,B,Ns,Hp,D] -> heads [h0, h0+P*Hp) of x_seq
        from ._lib import check, lib
        import ctypes as C
        P, B, Ns, Hp, D = recv.shape
        H = x_seq.shape[2]
        for t in (recv, x_seq):
            if not (t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous()):
                raise ValueError("Ulysses relayout needs contiguous bf16 CUDA tensors")
        check(lib.mod_ulysses_head_unpack_heads(C.c_void_p(recv.data_ptr()), C.c_void_p(x_seq.data_ptr()), B, Ns, Hp,
                                                D, P, H, h0,
                                                C.c_void_p(torch.cuda.current_stream(recv.device).cuda_stream)))
        return x_seq


KERNELS = KernelRelayout()


def _all_to_all(recv: torch.Tensor, send: torch.Tensor, group=None, async_op: bool = False):
    """all_to_all_single over equal per-peer chunks.  NCCL (the B200 path) exchanges the device tensors
    directly over NVLink; gloo (CPU-only collectives: the multi-process tests on one GPU) stages through
    host memory."""
    if dist.get_backend(group) == "gloo" and send.is_cuda:
        r_h = torch.empty(recv.shape, dtype=recv.dtype)
        dist.all_to_all_single(r_h, send.cpu(), group=group)
        recv.copy_(r_h)
        return None
    return dist.all_to_all_single(recv, send, group=group, async_op=async_op)


def seq_to_heads(x_seq: torch.Tensor, group=None, relayout=None, out=None) -> torch.Tensor:
    """Ulysses forward all-to-all: sequence shard [B, N/P, H, D] -> head shard [B, H/P, N, D] (contiguous).

    Rank r holds tokens [r*N/P, (r+1)*N/P) of every head; afterwards it holds every token of heads
    [r*H/P, (r+1)*H/P).  pack kernel -> one all_to_all_single -> unpack kernel (at P = 1 the unpack
    alone is the transpose).  ``out`` receives the head shard (the kernel relayout writes it in place);
    ``relayout`` swaps the pack/unpack implementation (the CPU gloo tests)."""
    rl = relayout or KERNELS
    P = _world(group)
    B, Ns, H, D = x_seq.shape
    if H % P:
        raise ValueError(f"heads={H} not divisible by world size {P}")
    unpack = (lambda t: rl.seq_unpack(t, out=out)) if out is not None else rl.seq_unpack
    if P == 1:
        return unpack(x_seq.reshape(1, B, Ns, H, D))
    send = rl.seq_pack(x_seq, P)                   # [P (destination = head group), B, Ns, Hp, D]
    recv = torch.empty_like(send)                  # [P (source = sequence chunk), B, Ns, Hp, D]
    _all_to_all(recv, send, group)
    return unpack(recv)


def heads_to_seq(x_head: torch.Tensor, group=None, relayout=None, out=None) -> torch.Tensor:
    """Ulysses inverse all-to-all: head shard [B, H/P, N, D] -> sequence shard [B, N/P, H, D]."""
    rl = relayout or KERNELS
    P = _world(group)
    B, Hp, N, D = x_head.shape
    if N % P:
        raise ValueError(f"tokens={N} not divisible by world size {P}")
    if P == 1:
        dst = None if out is None else out.view(1, B, N, Hp, D)
        send = rl.head_pack(x_head, 1, out=dst) if dst is not None else rl.head_pack(x_head, 1)
        return send.reshape(B, N, Hp, D)
    send = rl.head_pack(x_head, P)                 # [P (destination = sequence chunk), B, Ns, Hp, D]
    recv = torch.empty_like(send)                  # [P (source = head group), B, Ns, Hp, D]
    _all_to_all(recv, send, group)
    return rl.head_unpack(recv, out=out) if out is not None else rl.head_unpack(recv)


def ulysses_chunk_heads(H: int, P: int, chunks: int, rank: int) -> list[int]:
    """Global heads a rank owns in the chunked exchange: chunk c covers heads [c*H/C, (c+1)*H/C) and
    rank r takes the r-th of its P sub-blocks, [c*H/C + r*H/(C*P), +H/(C*P))."""
    if H % (chunks * P):
        raise ValueError(f"heads={H} not divisible by chunks*P={chunks * P}")
    hc, hl = H // chunks, H // (chunks * P)
    return [c * hc + rank * hl + i for c in range(chunks) for i in range(hl)]


class UlyssesChunkPipeline:
    """Sequence-sharded step with the Ulysses all-to-alls overlapped with the hot path, by head chunks.

    Rank r holds x_seq = tokens [r*N/P, (r+1)*N/P) of all H heads ([B, N/P, H, D] for Q, K, V).  The H
    heads are cut into C chunks of H/C; for chunk c the pack kernel gathers the chunk's heads, one
    all_to_all_single (NCCL over NVLink) delivers to each rank its H/(C*P) heads of the chunk with every
    token, the unpack kernel lays them out [B, H/(C*P), N, D], the caller's per-head step runs on them
    (``step_fn(plan, c, q, k, v, o)``), and the inverse exchange writes O back into the chunk's heads of
    o_seq.  Three streams: the forward exchange of chunk c+1 and the inverse exchange of chunk c-1 run
    while chunk c computes; head-shard buffers are double-buffered and their reuse is event-ordered.
    Every step of MOD-DiT is per head, so the chunking changes no result bit.
    """

    def __init__(self, layout, chunks: int, group=None, **plan_kw):
        import dataclasses
        from .plan import LayoutSpec, Plan
        spec = LayoutSpec.from_any(layout)
        self.P = _world(group)
        self.group = group
        self.rank = dist.get_rank(group) if self.P > 1 else 0
        H = spec.heads
        if H % (chunks * self.P):
            raise ValueError(f"heads={H} not divisible by chunks*P={chunks * self.P}")
        if spec.tokens % self.P:
            raise ValueError(f"tokens={spec.tokens} not divisible by P={self.P}")
        self.spec, self.chunks = spec, chunks
        self.hc, self.hl = H // chunks, H // (chunks * self.P)
        self.plan = Plan(dataclasses.replace(spec, heads=self.hl), **plan_kw)
        dev = torch.device(f"cuda:{self.plan.device}")
        B, N, D = spec.batch, spec.tokens, spec.head_dim
        Ns = N // self.P
        hshape = (B, self.hl, N, D)
        cshape = (self.P, B, Ns, self.hl, D)
        mk = lambda shape: torch.empty(shape, dtype=torch.bfloat16, device=dev)
        self.qh = [[mk(hshape) for _ in range(3)] for _ in range(2)]     # [slot][q, k, v] head shards
        self.oh = [mk(hshape) for _ in range(2)]
        self.send = [[mk(cshape) for _ in range(3)] for _ in range(2)]
        self.recv = [[mk(cshape) for _ in range(3)] for _ in range(2)]
        self.osend = [mk(cshape) for _ in range(2)]
        self.orecv = [mk(cshape) for _ in range(2)]
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
        self._free = [None, None]     # slot's head shards / send buffers reusable (compute of its last chunk done)
        self._odone = [None, None]    # slot's O shard / osend reusable (inverse exchange of its last chunk done)

    def heads(self, c: int) -> list[int]:
        """Global heads of chunk c that this rank computes."""
        base = c * self.hc + self.rank * self.hl
        return list(range(base, base + self.hl))

    def _issue_in(self, c, xs, start):
        rl, P, sl = KERNELS, self.P, c % 2
        with torch.cuda.stream(self.s_in):
            self.s_in.wait_event(start)
            if self._free[sl] is not None:
                self.s_in.wait_event(self._free[sl])
            for x, snd, rcv, dst in zip(xs, self.send[sl], self.recv[sl], self.qh[sl]):
                rl.seq_pack_heads(x, c * self.hc, self.hc, P, out=snd)
                if P > 1:
                    w = _all_to_all(rcv, snd, self.group, async_op=True)
                    if w is not None:
                        w.wait()
                    rl.seq_unpack(rcv, out=dst)
                else:
                    rl.seq_unpack(snd, out=dst)
            arrived = torch.cuda.Event()
            arrived.record(self.s_in)
        return arrived

    def _issue_compute_out(self, c, arrived, o_seq, step_fn):
        rl, P, sl = KERNELS, self.P, c % 2
        with torch.cuda.stream(self.s_comp):
            self.s_comp.wait_event(arrived)
            if self._odone[sl] is not None:
                self.s_comp.wait_event(self._odone[sl])
            q, k, v = self.qh[sl]
            step_fn(self.plan, c, q, k, v, self.oh[sl])
            computed = torch.cuda.Event()
            computed.record(self.s_comp)
            self._free[sl] = computed
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(computed)
            rl.head_pack(self.oh[sl], P, out=self.osend[sl])
            if P > 1:
                w = _all_to_all(self.orecv[sl], self.osend[sl], self.group, async_op=True)
                if w is not None:
                    w.wait()
                rl.head_unpack_heads(self.orecv[sl], o_seq, c * self.hc)
            else:
                rl.head_unpack_heads(self.osend[sl], o_seq, c * self.hc)
            od = torch.cuda.Event()
            od.record(self.s_out)
            self._odone[sl] = od

    def run(self, q_seq, k_seq, v_seq, o_seq, step_fn):
        """One step: ``q_seq, k_seq, v_seq`` [B, N/P, H, D] are this rank's sequence shards, ``o_seq`` receives
        O in the same layout.  The forward exchange of chunk c+1 is issued BEFORE the inverse exchange of
        chunk c, so that (NCCL runs a communicator's collectives in issue order) it overlaps chunk c's
        compute.  Returns after enqueueing; the caller's stream waits for the last inverse exchange."""
        caller = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(caller)
        xs = (q_seq, k_seq, v_seq)
        arrived = self._issue_in(0, xs, start)
        for c in range(self.chunks):
            nxt = self._issue_in(c + 1, xs, start) if c + 1 < self.chunks else None
            self._issue_compute_out(c, arrived, o_seq, step_fn)
            arrived = nxt
        for sl in range(min(2, self.chunks)):
            caller.wait_event(self._odone[sl])
