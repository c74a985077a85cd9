"""Multi-GPU plumbing of the hot path: head partitioning and the Ulysses all-to-all.

Every step of MOD-DiT is per (batch, head) -- statistics, fit, prediction, update and attention
(§4.1 P:202 "We process each attention head independently"; §5.3 P:439-442 the layer mask
is the concatenation of per-head masks).  The path therefore shards by heads with no collective
on the data path.  A collective appears only when the activations arrive sequence-sharded (the
usual DiT sequence parallelism): then a Ulysses all-to-all turns [B, N/P, H, D] sequence shards
into [B, H/P, N, D] head shards before the hot path and back afterwards.  The all-to-all runs on
NCCL through torch.distributed (NVLink 5 / NVSwitch on a B200 node); gloo is used by the CPU tests.
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


def seq_to_heads(x_seq: torch.Tensor, group=None) -> torch.Tensor:
    """Ulysses forward all-to-all: sequence shard [B, N/P, H, D] -> head shard [B, H/P, N, D] (contiguous).

    Rank r holds tokens [r*N/P, (r+1)*N/P) of every head; afterwards it holds every token of heads
    [r*H/P, (r+1)*H/P).  One all_to_all_single per tensor (a local permute when P = 1)."""
    P = _world(group)
    if P == 1:
        return x_seq.permute(0, 2, 1, 3).contiguous()
    B, Ns, H, D = x_seq.shape
    if H % P:
        raise ValueError(f"heads={H} not divisible by world size {P}")
    Hp = H // P
    # send buffer: [P (destination = head group), B, Ns, Hp, D]
    send = x_seq.reshape(B, Ns, P, Hp, D).permute(2, 0, 1, 3, 4).contiguous()
    recv = torch.empty_like(send)                     # [P (source = sequence chunk), B, Ns, Hp, D]
    dist.all_to_all_single(recv, send, group=group)
    return recv.permute(1, 3, 0, 2, 4).reshape(B, Hp, P * Ns, D).contiguous()


def heads_to_seq(x_head: torch.Tensor, group=None) -> torch.Tensor:
    """Ulysses inverse all-to-all: head shard [B, H/P, N, D] -> sequence shard [B, N/P, H, D]."""
    P = _world(group)
    if P == 1:
        return x_head.permute(0, 2, 1, 3).contiguous()
    B, Hp, N, D = x_head.shape
    if N % P:
        raise ValueError(f"tokens={N} not divisible by world size {P}")
    Ns = N // P
    # send buffer: [P (destination = sequence chunk), B, Ns, Hp, D]
    send = x_head.reshape(B, Hp, P, Ns, D).permute(2, 0, 3, 1, 4).contiguous()
    recv = torch.empty_like(send)                     # [P (source = head group), B, Ns, Hp, D]
    dist.all_to_all_single(recv, send, group=group)
    return recv.permute(1, 2, 0, 3, 4).reshape(B, Ns, P * Hp, D).contiguous()
