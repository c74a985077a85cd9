"""Quantized (INT8 QK / FP8 PV) vs bf16 K4 at a config's shape with structured masks."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic as syn
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _masks import structured_csr
import paper_2601_11641_b200 as M
from bench import attn_flops

w = syn.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hunyuanvideo-720p"]
REPS = int(os.environ.get("REPS", "10"))
P = M.Plan(w)
q, k, v = syn.family_s(w, step=12, device="cuda")
rp, ci = structured_csr(P, w)
nnz = float(rp[..., -1].sum().item())
density = nnz / (w.batch * w.heads * P.n * P.n)
fl = attn_flops(rp.cpu().numpy(), ci.cpu().numpy(), w.tokens, w.block, w.head_dim)
qb = P.quantize_qkv(q, k, v)
o8, l8 = P.block_sparse_attn_fwd_q8(qb, rp, ci)
ob, lb = P.block_sparse_attn_fwd(q, k, v, rp, ci)
torch.cuda.synchronize()
d = (o8.float() - ob.float()).abs()
res = {"config": w.name, "density": round(density, 4), "tflop": round(fl / 1e12, 3),
       "q8_vs_bf16_max_abs": round(d.max().item(), 4), "q8_vs_bf16_mean_abs": round(d.mean().item(), 6),
       "lse_max_abs": round((l8 - lb).abs().max().item(), 5)}
def t(fn):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(REPS):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / REPS
res["quantize_ms"] = round(t(lambda: P.quantize_qkv(q, k, v, out=qb)), 3)
res["attn_q8_ms"] = round(t(lambda: P.block_sparse_attn_fwd_q8(qb, rp, ci, out=o8, lse=l8)), 3)
res["attn_bf16_ms"] = round(t(lambda: P.block_sparse_attn_fwd(q, k, v, rp, ci, out=ob, lse=lb)), 3)
res["q8_tflops_equiv"] = round(fl / res["attn_q8_ms"] / 1e9, 1)
res["bf16_tflops"] = round(fl / res["attn_bf16_ms"] / 1e9, 1)
res["speedup_attn"] = round(res["attn_bf16_ms"] / res["attn_q8_ms"], 3)
res["speedup_with_quantize"] = round(res["attn_bf16_ms"] / (res["attn_q8_ms"] + res["quantize_ms"]), 3)
print(json.dumps(res))
