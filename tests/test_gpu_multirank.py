"""Multi-rank execution of one Alg.-1 re-estimation step on ONE GPU with 2 processes and
the gloo backend, against the single-rank run:

  * head-parallel: rank r owns heads [2r, 2r+2) of a 4-head layout (the bench's head partitioning);
  * chunked Ulysses (BASELINE config 5): each rank holds the sequence shard [r N/2, (r+1) N/2) of every
    head, UlyssesChunkPipeline exchanges head chunks (pack kernel -> all-to-all -> unpack kernel), runs
    the step on its heads of each chunk and exchanges O back into the sequence shard.

Every step of MOD-DiT is per head ("We process each attention head independently"; P:439-442 the
layer mask is the concatenation of per-head masks), so O, lse, the predicted CSR masks, the Eq. 5
history and the refit intensities must be BITWISE identical to the single-rank run.  gloo stages the
all-to-all through host memory (NCCL exchanges device buffers on a B200 node); every other step runs the
same libmoddit kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch

import synthetic as syn

pytestmark = pytest.mark.gpu

W = syn.Workload("mr-small", 1, 4, 128, 40, 3, 20, 19, 128)     # N = 1180, 10 blocks, ragged tail 28
K = 8
T_PREV, T_CURR, T_P = 11, 12, 22


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _warm(P, heads):
    """Warm-up of Alg. 1 for `heads`: statistics at t = 11, 12, fits, keep, history."""
    q1, k1, _ = syn.family_s_heads(W, heads, step=T_PREV, device="cuda")
    q, k, v = syn.family_s_heads(W, heads, step=T_CURR, device="cuda")
    W1, W2 = P.collect_block_stats(q1, k1), P.collect_block_stats(q, k)
    x1, x2 = P.fit_mixture(W1), P.fit_mixture(W2)
    keep = P.keep_frames(x1, x2)
    return dict(x1=x1, x2=x2, keep=keep, hist=W2.clone())


def _step(P, st, sl, q, k, v, o=None):
    """The re-estimation step on heads `sl` of the state: predict (Eq. 6/7) -> attention -> fresh
    statistic -> Eq. 5 update + refit + roll."""
    x1, x2, keep, hist = st["x1"][:, sl], st["x2"][:, sl], st["keep"][:, sl], st["hist"][:, sl]
    rp, ci = P.predict_block_mask(x1, x2, T_PREV, T_CURR, T_P, keep, top_k=K)
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o)
    Wf = P.collect_block_stats(q, k)
    P.update_online_mask(Wf, rp, ci, hist, x1, x2)
    return o, lse, rp, ci


def _np(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy() if t.dtype == torch.bfloat16 else t.cpu().numpy()


def _reference():
    from paper_2601_11641_b200 import Plan
    P = Plan(W, top_k=1, tau_e=0.0)
    heads = list(range(W.heads))
    st = _warm(P, heads)
    q, k, v = syn.family_s_heads(W, heads, step=T_CURR, device="cuda")
    o, lse, rp, ci = _step(P, st, slice(None), q, k, v)
    torch.cuda.synchronize()
    return {h: dict(o=_np(o[:, h]), lse=_np(lse[:, h]), rp=_np(rp[:, h]), ci=_np(ci[:, h]),
                    hist=_np(st["hist"][:, h]), x=_np(st["x2"][:, h])) for h in heads}


def _worker(rank, ws, port, mode, q_out):
    try:
        _work(rank, ws, port, mode, q_out)
    except BaseException as e:   # report instead of leaving the parent waiting on the queue
        import traceback
        q_out.put((rank, {"error": traceback.format_exc()}))
        raise


def _work(rank, ws, port, mode, q_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2601_11641_b200 import Plan
        from paper_2601_11641_b200.parallel import UlyssesChunkPipeline, head_range, ulysses_chunk_heads
        res = {}
        if mode == "heads":
            h0, h1 = head_range(W.heads, ws, rank)
            heads = list(range(h0, h1))
            P = Plan(W.with_heads(len(heads)), top_k=1, tau_e=0.0)
            st = _warm(P, heads)
            q, k, v = syn.family_s_heads(W, heads, step=T_CURR, device="cuda")
            o, lse, rp, ci = _step(P, st, slice(None), q, k, v)
            torch.cuda.synchronize()
            for i, h in enumerate(heads):
                res[h] = dict(o=_np(o[:, i]), lse=_np(lse[:, i]), rp=_np(rp[:, i]), ci=_np(ci[:, i]),
                              hist=_np(st["hist"][:, i]), x=_np(st["x2"][:, i]))
        else:
            chunks = 2
            heads = ulysses_chunk_heads(W.heads, ws, chunks, rank)
            pipe = UlyssesChunkPipeline(W, chunks, top_k=1, tau_e=0.0)
            assert [h for c in range(chunks) for h in pipe.heads(c)] == heads
            st = _warm(Plan(W.with_heads(len(heads)), top_k=1, tau_e=0.0), heads)   # state of this rank's heads
            Ns = W.tokens // ws
            qs, ks, vs = syn.family_s_seq_shard(W, rank * Ns, (rank + 1) * Ns, step=T_CURR, device="cuda")
            os_ = torch.empty_like(qs)
            per_chunk = {}

            def step_fn(plan, c, q, k, v, o):
                sl = slice(c * pipe.hl, (c + 1) * pipe.hl)
                per_chunk[c] = _step(plan, st, sl, q, k, v, o=o)

            pipe.run(qs, ks, vs, os_, step_fn)
            torch.cuda.synchronize()
            res["o_seq"] = _np(os_)
            for c in range(chunks):
                _, lse, rp, ci = per_chunk[c]
                for i, h in enumerate(pipe.heads(c)):
                    j = c * pipe.hl + i
                    res[h] = dict(lse=_np(lse[:, i]), rp=_np(rp[:, i]), ci=_np(ci[:, i]),
                                  hist=_np(st["hist"][:, j]), x=_np(st["x2"][:, j]))
        q_out.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["heads", "ulysses"])
def test_two_ranks_on_one_gpu_match_single_rank(mode):
    import torch.multiprocessing as mp
    ref = _reference()
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, mode, q)) for r in range(ws)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(ws))
    for r, res in got.items():
        assert "error" not in res, res.get("error")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    Ns = W.tokens // ws
    for r, res in got.items():
        for h, d in res.items():
            if h == "o_seq":
                # [B, Ns, H, D] sequence shard of O vs the reference heads' token range
                for hh in range(W.heads):
                    assert np.array_equal(d[:, :, hh], ref[hh]["o"][:, r * Ns:(r + 1) * Ns]), (mode, r, hh)
                continue
            for key, val in d.items():
                if key == "ci":   # CSR capacity beyond nnz is unspecified: compare the lists themselves
                    nnz = int(d["rp"][..., -1].max())
                    assert np.array_equal(val[..., :nnz], ref[h][key][..., :nnz]), (mode, r, h, key)
                    continue
                assert np.array_equal(val, ref[h][key]), (mode, r, h, key)
    covered = sorted(h for res in got.values() for h in res if h != "o_seq")
    assert covered == list(range(W.heads))
