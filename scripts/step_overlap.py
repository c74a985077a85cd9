"""The bench's re-estimation step (K2b predict -> K4 -> K1 -> K3) with K1 serial after K4 (bench.py) or on a
second stream concurrent with K4 (K1 reads the step's Q, K only; K3 joins both).  CUDA-event time per step.
  python scripts/step_overlap.py [config] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synthetic as syn
import paper_2601_11641_b200 as M

cfg = sys.argv[1] if len(sys.argv) > 1 else "hunyuanvideo-720p"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
K = {"cogvideox-5b": 12, "wan2.1-14b-720p": 96}.get(cfg, 164)
w = syn.CONFIGS[cfg]
P = M.Plan(w, top_k=1)
q1, k1, _ = syn.family_s(w, step=11, device="cuda")
W1 = P.collect_block_stats(q1, k1)
del q1, k1
q, k, v = syn.family_s(w, step=12, device="cuda")
W2 = P.collect_block_stats(q, k)
x1, x2 = P.fit_mixture(W1), P.fit_mixture(W2)
keep = P.keep_frames(x1, x2)
rp, ci = P.predict_block_mask(x1, x2, 11, 12, 22, keep, top_k=K)
o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
Wf, hist = W2.clone(), W1.clone()
xp, xc = x1.clone(), x2.clone()
main = torch.cuda.current_stream()
side = torch.cuda.Stream()
# K1 needs its own workspace when it runs beside K4 (Plan.workspace(stream)); K4 itself does not use one
ws_side = None


def serial():
    P.predict_block_mask(x1, x2, 11, 12, 22, keep, top_k=K, out=(rp, ci))
    P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
    P.collect_block_stats(q, k, out=Wf)
    P.update_online_mask(Wf, rp, ci, hist, xp, xc)


def overlapped():
    P.predict_block_mask(x1, x2, 11, 12, 22, keep, top_k=K, out=(rp, ci))
    ev0 = torch.cuda.Event()
    ev0.record(main)
    side.wait_event(ev0)
    with torch.cuda.stream(side):
        P.collect_block_stats(q, k, out=Wf)
    P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
    ev1 = torch.cuda.Event()
    ev1.record(side)
    main.wait_event(ev1)
    P.update_online_mask(Wf, rp, ci, hist, xp, xc)


def overlapped_k13():   # K1 and K3 both on the side stream beside K4 (K3 needs only K1 and the mask)
    P.predict_block_mask(x1, x2, 11, 12, 22, keep, top_k=K, out=(rp, ci))
    side.wait_stream(main)
    with torch.cuda.stream(side):
        P.collect_block_stats(q, k, out=Wf)
        P.update_online_mask(Wf, rp, ci, hist, xp, xc)
    P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
    main.wait_stream(side)


res = {"config": cfg}
for _ in range(max(10, 3 * reps)):   # warm up to the power / thermal steady state
    serial()
times = {"serial": [], "overlapped": [], "overlapped_k13": []}
for r in range(4):   # alternating blocks
    for name, fn in (("serial", serial), ("overlapped", overlapped), ("overlapped_k13", overlapped_k13)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for _ in range(reps):
            fn()
        e1.record(main)
        torch.cuda.synchronize()
        times[name].append(round(e0.elapsed_time(e1) / reps, 4))
for name, t in times.items():
    res[name + "_ms"] = t
    res[name + "_mean_ms"] = round(sum(t) / len(t), 4)
res["gain"] = round(res["serial_mean_ms"] / res["overlapped_mean_ms"] - 1, 4)
res["gain_k13"] = round(res["serial_mean_ms"] / res["overlapped_k13_mean_ms"] - 1, 4)
print(json.dumps(res))
