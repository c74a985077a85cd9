"""HeadChunkPipeline (host-resident activations, head chunks overlapped on three streams) against the
same Plan calls run serially on the whole problem.  Every step of the hot path is per (b, h)
(SURVEY §8(e)), so the pipelined step must reproduce the serial one BIT FOR BIT: outputs on the
host, the updated history map and the rolled intensities."""
import numpy as np
import pytest
import torch

import synthetic as syn

pytestmark = pytest.mark.gpu

W = syn.Workload("pipe-small", 1, 6, 128, 40, 3, 20, 19, 128)   # N=1180, n=10, ragged tail


@pytest.mark.parametrize("chunks", [1, 3, 6])
def test_pipeline_matches_serial_step(chunks):
    from paper_2601_11641_b200 import Plan
    from paper_2601_11641_b200.pipeline import HeadChunkPipeline

    q, k, v = syn.family_s(W, device="cuda")
    P = Plan(W, top_k=4)
    W1 = P.collect_block_stats(*syn.family_s(W, step=1, device="cuda")[:2])
    W2 = P.collect_block_stats(q, k)
    x_prev0, x_curr0 = P.fit_mixture(W1), P.fit_mixture(W2)
    keep = P.keep_frames(x_prev0, x_curr0)

    def state():
        return W2.clone(), x_prev0.clone(), x_curr0.clone()

    # serial reference: two steps on the whole problem
    hist_r, xp_r, xc_r = state()
    outs_r = []
    for t in (22, 23):
        rp, ci = P.predict_block_mask(x_prev0, x_curr0, 11, 12, t, keep)
        o, _ = P.block_sparse_attn_fwd(q, k, v, rp, ci)
        P.update_online_mask(P.collect_block_stats(q, k), rp, ci, hist_r, xp_r, xc_r)
        outs_r.append(o.cpu())

    # pipelined: host-resident inputs, head chunks on three streams
    pipe = HeadChunkPipeline(W, chunks, top_k=4)
    hist, xp, xc = state()
    rp, ci = P.empty_mask()
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device="cuda")
    Wf = P.empty_stats()
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    for t, o_ref in zip((22, 23), outs_r):
        ho = torch.zeros_like(hq).pin_memory()

        def step(plan, c, qc, kc, vc, oc):
            hs = pipe.heads(c)
            plan.predict_block_mask(x_prev0[:, hs], x_curr0[:, hs], 11, 12, t, keep[:, hs], out=(rp[:, hs], ci[:, hs]))
            plan.block_sparse_attn_fwd(qc, kc, vc, rp[:, hs], ci[:, hs], out=oc, lse=lse[:, hs])
            plan.collect_block_stats(qc, kc, out=Wf[:, hs])
            plan.update_online_mask(Wf[:, hs], rp[:, hs], ci[:, hs], hist[:, hs], xp[:, hs], xc[:, hs])

        pipe.run(hq, hk, hv, ho, step)
        torch.cuda.synchronize()
        assert torch.equal(ho, o_ref)
    assert torch.equal(hist, hist_r)
    assert np.array_equal(xp.cpu().numpy(), xp_r.cpu().numpy())
    assert np.array_equal(xc.cpu().numpy(), xc_r.cpu().numpy())


def test_pipeline_rejects_bad_chunking():
    from paper_2601_11641_b200.pipeline import HeadChunkPipeline
    with pytest.raises(ValueError, match="not divisible"):
        HeadChunkPipeline(W, 4)
