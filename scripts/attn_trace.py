"""Dump the clock64 event trace of CTA 1000 (MOD_ATTN_DEBUG=16|x) at the Hunyuan shape."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic as syn
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _masks import structured_csr
import paper_2601_11641_b200 as M
w = syn.CONFIGS[sys.argv[1]] if len(sys.argv) > 1 else syn.HUNYUAN
P = M.Plan(w)
q, k, v = syn.family_r(w, device="cuda")
rp, ci = structured_csr(P, w)
nnz = float(rp[..., -1].sum().item())
density = nnz / (w.batch * w.heads * P.n * P.n)
o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci); torch.cuda.synchronize()
buf = (ctypes.c_longlong * (5 * 4096 * 2))()
M.lib.mod_debug_attn_trace(buf, 5 * 4096 * 2)
o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci); torch.cuda.synchronize()
M.lib.mod_debug_attn_trace(buf, 5 * 4096 * 2)
ev = sorted((buf[2 * i], buf[2 * i + 1] >> 32, buf[2 * i + 1] & 0xffffffff) for i in range(5 * 4096) if buf[2 * i])
n = len(ev)
t0 = ev[0][0]
names = {1: "P:k_empty", 2: "P:v_empty", 10: "M:k_full", 11: "M:S_issued", 12: "M:p_full", 13: "M:v_full", 14: "M:PV_issued",
         20: "S0:s_full", 21: "S1:s_full", 30: "S0:exp_done", 31: "S1:exp_done", 40: "S0:p_arrive", 41: "S1:p_arrive", 50: "S0:ld_done", 51: "S1:ld_done", 60: "S0:max_xchg", 61: "S1:max_xchg"}
with open("gpurun_out/trace.txt", "w") as f:
    for t, tag, j in ev:
        f.write(f"{t - t0:9d} {names.get(tag, tag):14s} j={j}\n")
print("events", n, "span", ev[-1][0] - t0, "list length", int((rp[0, 1000 // P.n, 1000 % P.n + 1] - rp[0, 1000 // P.n, 1000 % P.n]).item()), "n", P.n)
