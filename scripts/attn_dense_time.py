"""Time K4 with the all-ones list (dense) and a structured sparse list at the Hunyuan shape (bring-up)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synthetic as syn
import paper_2601_11641_b200 as M
w = syn.HUNYUAN.with_heads(int(os.environ.get("HEADS", "4")))
P = M.Plan(w)
q, k, v = syn.family_r(w, device="cuda")
rp, ci = P.dense_mask()
o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1); fl = 4.0 * w.head_dim * w.tokens ** 2 * w.heads
print(json.dumps({"lib": M.LIB_PATH, "dense_ms": ms, "dense_tflops": fl / ms / 1e9}))
