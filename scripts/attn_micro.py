"""K4 micro-timing at the Hunyuan shape with structured masks (bring-up experiments).
MOD_ATTN_DEBUG=1: softmax skipped (MMA+TMA only); =2: K/V TMA skipped; =3 both."""
import os, sys, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic as syn
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _masks import structured_csr
import paper_2601_11641_b200 as M
from bench import attn_flops

w = syn.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hunyuanvideo-720p"]
P = M.Plan(w)
q, k, v = syn.family_r(w, device="cuda")
rp, ci = structured_csr(P, w)
nnz = float(rp[..., -1].sum().item())
density = nnz / (w.batch * w.heads * P.n * P.n)
fl = attn_flops(rp.cpu().numpy(), ci.cpu().numpy(), w.tokens, w.block, w.head_dim)
o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
torch.cuda.synchronize()
import threading, pynvml
pynvml.nvmlInit(); hnd = pynvml.nvmlDeviceGetHandleByIndex(0); clk = []; pw = []; stop = threading.Event()
def samp():
    while not stop.is_set():
        clk.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)); pw.append(pynvml.nvmlDeviceGetPowerUsage(hnd) / 1000.0); stop.wait(0.01)
th = threading.Thread(target=samp); th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
REPS = int(os.environ.get("REPS", "5"))
for _ in range(REPS):
    P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
e1.record(); torch.cuda.synchronize(); stop.set(); th.join()
ms = e0.elapsed_time(e1) / REPS
mhz = float(np.median(clk)) if clk else float("nan")
iters_per_sm = nnz / 148
print(json.dumps({"lib": os.environ.get("MODDIT_LIB_OVERRIDE", "default"), "dbg": os.environ.get("MOD_ATTN_DEBUG", "0"),
                  "density": round(density, 4), "ms": round(ms, 3), "tflops": round(fl / ms / 1e9, 1),
                  "sm_mhz": mhz, "watts": round(float(np.median(pw[len(pw)//3:])), 0) if pw else None, "mhz_late": float(np.median(clk[len(clk)//3:])) if clk else None, "cycles_per_block_iter": round(ms * 1e-3 * mhz * 1e6 / iters_per_sm, 1)}))
