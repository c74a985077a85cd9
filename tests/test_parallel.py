"""Head partitioning and the Ulysses all-to-all on CPU with gloo, world size 2 and 4."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_11641_b200.parallel import head_range, heads_to_seq, lpt_head_assignment, seq_to_heads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class TorchRelayout:
    """Test-side reference of the pack / unpack maps (include/moddit.h mod_ulysses_*), in torch, so
    that the all-to-all plumbing runs on CPU with gloo.  The CUDA kernels are pinned to the same maps
    in tests/test_gpu_ulysses.py."""

    @staticmethod
    def seq_pack(x_seq, P):
        B, Ns, H, D = x_seq.shape
        return x_seq.reshape(B, Ns, P, H // P, D).permute(2, 0, 1, 3, 4).contiguous()

    @staticmethod
    def seq_unpack(recv):
        P, B, Ns, Hp, D = recv.shape
        return recv.permute(1, 3, 0, 2, 4).reshape(B, Hp, P * Ns, D).contiguous()

    @staticmethod
    def head_pack(x_head, P):
        B, Hp, N, D = x_head.shape
        return x_head.reshape(B, Hp, P, N // P, D).permute(2, 0, 3, 1, 4).contiguous()

    @staticmethod
    def head_unpack(recv):
        P, B, Ns, Hp, D = recv.shape
        return recv.permute(1, 2, 0, 3, 4).reshape(B, Ns, P * Hp, D).contiguous()


def _worker(rank, ws, port, B, N, H, D, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        g = torch.Generator().manual_seed(0)
        full = torch.randn((B, N, H, D), generator=g)         # [B, N, H, D] activations, identical on all ranks
        Ns = N // ws
        x_seq = full[:, rank * Ns:(rank + 1) * Ns].contiguous()
        x_head = seq_to_heads(x_seq, relayout=TorchRelayout)
        h0, h1 = head_range(H, ws, rank)
        ref = full.permute(0, 2, 1, 3)[:, h0:h1].contiguous()  # [B, H/P, N, D]
        ok1 = torch.equal(x_head, ref)
        back = heads_to_seq(x_head, relayout=TorchRelayout)
        ok2 = torch.equal(back, x_seq)
        q.put((rank, ok1, ok2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 4])
def test_ulysses_roundtrip_gloo(ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, 2, 24, 8, 16, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] and r[2] for r in res), res


def test_head_range_and_lpt():
    assert [head_range(24, 8, r) for r in range(8)][-1] == (21, 24)
    with pytest.raises(ValueError):
        head_range(24, 5, 0)
    parts = lpt_head_assignment([5, 1, 4, 2, 3, 3], 2)
    assert sorted(sum(parts, [])) == list(range(6))
    loads = [sum([5, 1, 4, 2, 3, 3][h] for h in p) for p in parts]
    assert max(loads) - min(loads) <= 1


def test_relayout_reference_maps_p1():
    """At P = 1 the maps are the [B,N,H,D] <-> [B,H,N,D] transpose (what seq_to_heads returns)."""
    x = torch.randn(2, 5, 6, 8)
    assert torch.equal(seq_to_heads(x, relayout=TorchRelayout), x.permute(0, 2, 1, 3))
    assert torch.equal(heads_to_seq(x.permute(0, 2, 1, 3).contiguous(), relayout=TorchRelayout), x)


def test_family_s_head_lists_and_sequence_shards_are_the_full_tensor_bytes():
    """Per-rank generators (LPT head lists, Ulysses sequence shards) draw exactly the bytes of the full
    tensors, so multi-rank runs and the single-GPU run see the same inputs."""
    import synthetic as syn
    w = syn.Workload("t", 1, 4, 64, 10, 2, 4, 4, 64)
    q, k, v = syn.family_s(w, step=3)
    q2, k2, v2 = syn.family_s_heads(w, [2, 0], step=3)
    assert torch.equal(q2[:, 0], q[:, 2]) and torch.equal(k2[:, 1], k[:, 0]) and torch.equal(v2[:, 0], v[:, 2])
    qs, ks, vs = syn.family_s_seq_shard(w, 5, 20, step=3)
    for a, b in ((qs, q), (ks, k), (vs, v)):
        assert torch.equal(a, b.permute(0, 2, 1, 3)[:, 5:20])


def test_ulysses_chunk_heads_partition():
    from paper_2601_11641_b200.parallel import ulysses_chunk_heads
    for H, P, C in ((24, 2, 3), (24, 8, 3), (40, 4, 2), (4, 2, 2)):
        owned = [ulysses_chunk_heads(H, P, C, r) for r in range(P)]
        assert sorted(h for o in owned for h in o) == list(range(H))
        assert all(len(o) == H // P for o in owned)
