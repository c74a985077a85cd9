"""K4 pipeline trace (bring-up): run the default K4 of a -DMOD_K4_TRACE build on the bench workload
(Family S at HunyuanVideo 720p, the pipeline's K = 164 mask) and summarise
  * per-CTA clock64 / globaltimer spans: effective SM clock, cycles = a + b * blocks (fixed + per block)
  * the MMA thread's and one softmax warp's steady-state intervals per block (clock64 stamps).
  MODDIT_LIB_OVERRIDE=_variants/k4trace/libmoddit.so python scripts/k4_trace.py [config] [attn_kernel]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthetic as syn
import paper_2601_11641_b200 as M
from paper_2601_11641_b200 import _lib

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
for _ in range(3):
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
ncta = P.BH * P.n
fn = _lib.lib.mod_debug_k4_trace
fn.restype = ctypes.c_int
ev = np.zeros((8, 18, 512, 6), dtype=np.int64)
span = np.zeros((ncta, 4), dtype=np.int64)
fn(ev.ctypes.data_as(ctypes.c_void_p), span.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(ncta))
cyc, ns, t0, misc = span.T
L = misc & 0xffffffff
sm = misc >> 32
clock_ghz = cyc.sum() / ns.sum()
A = np.vstack([np.ones_like(L), L]).T.astype(float)
coef, *_ = np.linalg.lstsq(A, cyc.astype(float), rcond=None)
busy = np.zeros(148)
np.add.at(busy, sm, ns)
out = {"config": cfg, "kernel": P.attn_kernel_name(), "ms": round(ms, 3), "ctas": int(ncta),
       "blocks": int(L.sum()), "eff_clock_ghz": round(float(clock_ghz), 3),
       "cycles_fixed_per_cta": round(float(coef[0])), "cycles_per_block": round(float(coef[1]), 1),
       "sm_busy_frac": round(float(busy.mean() / (ms * 1e6)), 3)}
mma, smx = {}, {}
rows = []
for c in range(8):
    cta = c * 4096 + 1234
    if cta >= ncta:
        continue
    Lc = int(L[cta])
    if Lc < 40:
        continue
    J = range(6, min(Lc, 512) - 6)
    e = ev[c]
    d = lambda role, a, b: [e[role][j][b] - e[role][j][a] for j in J]
    per = lambda role, a: [e[role][j + 1][a] - e[role][j][a] for j in J]
    rows.append({"cta": cta, "L": Lc,
                 "mma_period": float(np.median(per(0, 0))), "mma_wait_v": float(np.median(d(0, 0, 1))),
                 "mma_wait_p": float(np.median(d(0, 1, 2))), "mma_pv_issue": float(np.median(d(0, 2, 3))),
                 "mma_s_issue": float(np.median(d(0, 3, 4))),
                 "sm_period": float(np.median(per(1, 0))), "sm_wait_s": float(np.median(d(1, 0, 1))),
                 "sm_ld": float(np.median(d(1, 1, 2))), "sm_exp": float(np.median(d(1, 2, 3))),
                 "sm_bar": float(np.median(d(1, 3, 4))), "sm_store_arrive": float(np.median(d(1, 4, 5)))})
out["traced"] = rows
print(json.dumps(out))
if os.environ.get("TIMELINE"):
    c = 0
    e = ev[c]
    base = e[0][20][0]
    nw = int(os.environ.get("NSMW", "8"))
    print("j | MMA: start, p_seen, pv_issued, s(j+3)_issued | P published by softmax warps 2..")
    for j in range(20, 27):
        m = [int(e[0][j][k] - base) for k in (0, 2, 3, 4)]
        pub = [int(e[1 + w][j][5] - base) for w in range(nw)]
        sseen = [int(e[1 + w][j][1] - base) for w in range(nw)]
        print(j, m, "pub", pub, "s_seen", sseen)
