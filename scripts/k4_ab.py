"""A/B of K4 schedules on the bench workload of each config (Family S, the predicted K-mask of the bench
step): CUDA-event time per launch and algorithmic TFLOP/s (4 D sum |I_i||I_j| over the listed blocks).
  python scripts/k4_ab.py [configs,comma-separated] [kernels,comma-separated] [reps]
Prints one JSON line per (config, kernel)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synthetic as syn
import paper_2601_11641_b200 as M

TOPK = {"cogvideox-5b": 12, "wan2.1-14b-720p": 96, "hunyuanvideo-720p": 164}
cfgs = (sys.argv[1] if len(sys.argv) > 1 else "cogvideox-5b,hunyuanvideo-720p").split(",")
kerns = (sys.argv[2] if len(sys.argv) > 2 else "default,wide").split(",")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dense = os.environ.get("DENSE", "0") == "1"

for cfg in cfgs:
    w = syn.CONFIGS[cfg]
    P0 = M.Plan(w, top_k=1)
    q1, k1, _ = syn.family_s(w, step=11, device="cuda")
    W1 = P0.collect_block_stats(q1, k1)
    del q1, k1
    q, k, v = syn.family_s(w, step=12, device="cuda")
    W2 = P0.collect_block_stats(q, k)
    x1, x2 = P0.fit_mixture(W1), P0.fit_mixture(W2)
    keep = P0.keep_frames(x1, x2)
    K = 10 ** 6 if dense else TOPK.get(cfg, 12)
    rp, ci = P0.predict_block_mask(x1, x2, 11, 12, 22, keep, top_k=K)
    n, N, blk, D = P0.n, P0.N, w.block, w.head_dim
    sizes = torch.clamp(N - torch.arange(n, device="cuda") * blk, max=blk).double()
    flops = 0.0
    rpl = rp.reshape(-1, n + 1).long()
    cil = ci.reshape(rpl.shape[0], -1).long()
    for h in range(rpl.shape[0]):
        cnt = rpl[h, 1:] - rpl[h, :-1]
        cols = cil[h, : int(rpl[h, -1])]
        rows = torch.repeat_interleave(torch.arange(n, device="cuda"), cnt)
        flops += float((sizes[rows] * sizes[cols]).sum()) * 4 * D
    nnz = float(rp[..., -1].sum())
    ref = None
    for kspec in kerns:
        kern, pool = kspec.split("+")[0], kspec.endswith("+pool")   # "default+pool": K4 with K1's fused means
        P = M.Plan(w, top_k=1, attn_kernel=kern)
        kw = {"pool": True} if pool else {}   # the fused-pool binding existed only in the experiment
        o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
        torch.cuda.synchronize()
        if ref is None:
            ref = o.float()
            dev = 0.0
        else:
            dev = (o.float() - ref).abs().max().item()
        for _ in range(2):
            P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse, **kw)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse, **kw)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"config": cfg, "kernel": P.attn_kernel_name() + ("+pool" if pool else ""), "ms": round(ms, 4),
                          "tflops": round(flops / ms / 1e9, 1), "nnz": nnz,
                          "sparsity": round(1 - nnz / (rp.shape[0] * rp.shape[1] * n * n), 4),
                          "max_dev_vs_first": dev}), flush=True)
    del q, k, v, W1, W2
    torch.cuda.empty_cache()
