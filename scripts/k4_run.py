"""Run K4 on the bench workload (Family S at a BASELINE shape, the pipeline's K = 164-style mask) REPS
times -- a short command for ncu captures of the attention kernel.
  python scripts/k4_run.py [config] [attn_kernel] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic as syn
import paper_2601_11641_b200 as M

cfg = sys.argv[1] if len(sys.argv) > 1 else "hunyuanvideo-720p"
w = syn.CONFIGS[cfg]
P = M.Plan(w, top_k=1, attn_kernel=sys.argv[2] if len(sys.argv) > 2 else "default")
q1, k1, _ = syn.family_s(w, step=11, device="cuda")
W1 = P.collect_block_stats(q1, k1)
del q1, k1
q, k, v = syn.family_s(w, step=12, device="cuda")
W2 = P.collect_block_stats(q, k)
x1, x2 = P.fit_mixture(W1), P.fit_mixture(W2)
keep = P.keep_frames(x1, x2)
rp, ci = P.predict_block_mask(x1, x2, 11, 12, 22, keep, top_k=int(os.environ.get("TOPK", "164")))
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
torch.cuda.synchronize()
print("ok", P.attn_kernel_name(), float(rp[..., -1].sum()))
