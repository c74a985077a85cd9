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


KERNELS = KernelRelayout()


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
    dist.all_to_all_single(recv, send, group=group)
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
    dist.all_to_all_single(recv, send, group=group)
    return rl.head_unpack(recv, out=out) if out is not None else rl.head_unpack(recv)
