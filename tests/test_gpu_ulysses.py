"""Ulysses relayout kernels (include/moddit.h mod_ulysses_*, BASELINE config 5) on one GPU.

All P ranks of a sequence-sharded layer are emulated on one device: every rank packs its shard with
the kernel, the all-to-all is replayed by indexing (rank r receives chunk r of every peer's send
buffer), and the unpacked head shard must equal the transpose of the full activation restricted to
the rank's heads -- bit for bit (a relayout moves bytes).  The packs are also compared with the torch
reference maps the CPU gloo tests use (tests/test_parallel.py)."""
import pytest
import torch

from test_parallel import TorchRelayout

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def PAR():
    from paper_2601_11641_b200 import parallel
    return parallel


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("D", [64, 128])
def test_relayout_roundtrip_emulated_ranks(PAR, P, D):
    B, H, N = 2, 24, 8 * 150 + 0          # N divisible by every P; heads by every P
    g = torch.Generator(device="cuda").manual_seed(P * 1000 + D)
    full = torch.randn((B, N, H, D), generator=g, device="cuda").to(torch.bfloat16)
    Ns, Hp = N // P, H // P
    K = PAR.KERNELS
    shards = [full[:, r * Ns:(r + 1) * Ns].contiguous() for r in range(P)]
    sends = [K.seq_pack(x, P) for x in shards]
    for x, s in zip(shards, sends):
        assert torch.equal(s, TorchRelayout.seq_pack(x, P))
    heads = []
    for r in range(P):
        recv = torch.stack([sends[p][r] for p in range(P)])          # the all-to-all, replayed
        xh = K.seq_unpack(recv)
        assert torch.equal(xh, full.permute(0, 2, 1, 3)[:, r * Hp:(r + 1) * Hp])
        heads.append(xh)
    sends2 = [K.head_pack(xh, P) for xh in heads]
    for xh, s in zip(heads, sends2):
        assert torch.equal(s, TorchRelayout.head_pack(xh, P))
    for r in range(P):
        recv = torch.stack([sends2[p][r] for p in range(P)])
        assert torch.equal(K.head_unpack(recv), shards[r])


def test_world_one_is_the_transpose(PAR):
    x = torch.randn((1, 1000, 6, 128), device="cuda").to(torch.bfloat16)
    xh = PAR.seq_to_heads(x)
    assert torch.equal(xh, x.permute(0, 2, 1, 3))
    assert torch.equal(PAR.heads_to_seq(xh), x)


def test_relayout_errors(PAR):
    import paper_2601_11641_b200 as M
    x = torch.zeros((1, 10, 6, 96), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(M.ModditError, match="head_dim=96"):
        PAR.KERNELS.seq_pack(x, 2)
    y = torch.zeros((1, 10, 6, 64), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(M.ModditError, match="not divisible"):
        PAR.KERNELS.seq_pack(y, 4)
    with pytest.raises(ValueError, match="CUDA"):
        PAR.KERNELS.seq_pack(y.cpu(), 2)


def test_out_argument_writes_in_place(PAR):
    x = torch.randn((1, 512, 6, 64), device="cuda").to(torch.bfloat16)
    dst = torch.empty((1, 6, 512, 64), device="cuda", dtype=torch.bfloat16)
    r = PAR.seq_to_heads(x, out=dst)
    assert r.data_ptr() == dst.data_ptr() and torch.equal(dst, x.permute(0, 2, 1, 3))
    back = torch.empty_like(x)
    r2 = PAR.heads_to_seq(dst, out=back)
    assert r2.data_ptr() == back.data_ptr() and torch.equal(back, x)


@pytest.mark.parametrize("P,C", [(1, 3), (2, 3), (4, 2), (8, 3)])
@pytest.mark.parametrize("D", [64, 128])
def test_head_chunk_relayouts_emulated_ranks(PAR, P, C, D):
    """mod_ulysses_seq_pack_heads / head_unpack_heads (the chunked pipeline's exchange): the chunk-c pack
    equals the whole-tensor pack of the chunk's heads, and unpacking every chunk's replayed exchange
    reconstructs every rank's sequence shard bit for bit, other heads untouched until written."""
    B, H, N = 1, 24, 8 * 150
    g = torch.Generator(device="cuda").manual_seed(P * 100 + C + D)
    full = torch.randn((B, N, H, D), generator=g, device="cuda").to(torch.bfloat16)
    Ns, Hc = N // P, H // C
    K = PAR.KERNELS
    shards = [full[:, r * Ns:(r + 1) * Ns].contiguous() for r in range(P)]
    outs = [torch.zeros_like(x) for x in shards]
    for c in range(C):
        h0 = c * Hc
        sends = [K.seq_pack_heads(x, h0, Hc, P) for x in shards]
        for x, s in zip(shards, sends):
            assert torch.equal(s, TorchRelayout.seq_pack(x[:, :, h0:h0 + Hc].contiguous(), P))
        head_shards = [K.seq_unpack(torch.stack([sends[p][r] for p in range(P)])) for r in range(P)]
        back = [K.head_pack(xh, P) for xh in head_shards]
        for r in range(P):
            K.head_unpack_heads(torch.stack([back[p][r] for p in range(P)]).contiguous(), outs[r], h0)
            untouched = outs[r][:, :, h0 + Hc:]
            assert torch.count_nonzero(untouched) == 0
    for x, o in zip(shards, outs):
        assert torch.equal(o, x)


def test_chunk_pipeline_single_rank_equals_unchunked(PAR):
    """UlyssesChunkPipeline at P = 1 (no process group): the chunked transposes + per-chunk hot path give
    the same O bits as running the plan on the whole head-major tensor."""
    import synthetic as syn
    from paper_2601_11641_b200 import Plan
    w = syn.Workload("cp-small", 1, 6, 128, 40, 3, 20, 19, 128)
    q, k, v = syn.family_s(w, step=12, device="cuda")
    P0 = Plan(w, top_k=1, tau_e=0.0)
    rp, ci = P0.dense_mask()
    o_ref, _ = P0.block_sparse_attn_fwd(q, k, v, rp, ci)
    pipe = PAR.UlyssesChunkPipeline(w, 3, top_k=1, tau_e=0.0)
    rpc, cic = pipe.plan.dense_mask()
    seq = [t.permute(0, 2, 1, 3).contiguous() for t in (q, k, v)]
    o_seq = torch.empty_like(seq[0])
    pipe.run(*seq, o_seq, lambda plan, c, qc, kc, vc, oc: plan.block_sparse_attn_fwd(qc, kc, vc, rpc, cic, out=oc))
    torch.cuda.synchronize()
    assert torch.equal(o_seq, o_ref.permute(0, 2, 1, 3))
