"""CUDA-event times of K1 (mod_collect_block_stats), K2a (mod_fit_mixture) and K3 (mod_update_online_mask) at a
config's shape on the bench's re-estimation inputs (Family S, the predicted K-mask).
  python scripts/time_k13.py [config] [top_k]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synthetic as syn
import paper_2601_11641_b200 as M

cfg = sys.argv[1] if len(sys.argv) > 1 else "hunyuanvideo-720p"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 164
w = syn.CONFIGS[cfg]
P = M.Plan(w, top_k=1)
q1, k1, _ = syn.family_s(w, step=11, device="cuda")
Wa = P.collect_block_stats(q1, k1)
del q1, k1
q, k, _ = syn.family_s(w, step=12, device="cuda")
Wb = P.collect_block_stats(q, k)
x1, x2 = P.fit_mixture(Wa), P.fit_mixture(Wb)
rp, ci = P.predict_block_mask(x1, x2, 11, 12, 22, P.keep_frames(x1, x2), top_k=K)
hist = Wa.clone()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


xp, xc = x1.clone(), x2.clone()
out = {"config": cfg, "library": os.environ.get("MODDIT_LIB_OVERRIDE", "in-tree"),
       "k1_ms": timed(lambda: P.collect_block_stats(q, k, out=Wb)),
       "k2a_fit_ms": timed(lambda: P.fit_mixture(Wb, out=x2)),
       "k3_update_ms": timed(lambda: P.update_online_mask(Wb, rp, ci, hist, xp, xc))}
out["k1_k3_ms"] = round(out["k1_ms"] + out["k3_update_ms"], 4)
print(json.dumps(out))
