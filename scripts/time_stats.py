"""Time K1 (pool + score) at a config's shape; run under ncu for per-kernel durations (bring-up)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synthetic as syn
import paper_2601_11641_b200 as M
w = syn.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hunyuanvideo-720p"]
P = M.Plan(w)
q, k, _ = syn.family_s(w, step=12, device="cuda")
W = P.collect_block_stats(q, k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(int(os.environ.get("REPS", "10"))):
    P.collect_block_stats(q, k, out=W)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"config": w.name, "k1_ms": e0.elapsed_time(e1) / int(os.environ.get("REPS", "10"))}))
