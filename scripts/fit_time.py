"""Times mod_fit_mixture (projection + RHS reduction + solve) at a config's layout, all heads."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synthetic as syn
import paper_2601_11641_b200 as M
w = syn.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hunyuanvideo-720p"]
P = M.Plan(w)
W = syn.random_stats(w.batch, w.heads, P.n, seed=1, device="cuda")
x = P.fit_mixture(W); torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); P.fit_mixture(W, out=x); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"lib": os.environ.get("MODDIT_LIB_OVERRIDE", "default"), "fit_ms": round(sorted(ts)[5], 4)}))
