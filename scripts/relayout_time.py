"""Bandwidth of the Ulysses relayout kernels at the Hunyuan 720p activation size (algorithmic bytes =
one read + one write of the tensor), P = 1 (transpose) and P = 8 (pack into 8 peer chunks)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_11641_b200.parallel import KERNELS
B, N, H, D = 1, 118800, 24, 128
x = torch.randn((B, N, H, D), device="cuda").to(torch.bfloat16)
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
for name, fn in (("seq_unpack P=1 (transpose)", lambda: KERNELS.seq_unpack(x.view(1, B, N, H, D))),
                 ("seq_pack P=8", lambda: KERNELS.seq_pack(x, 8)),
                 ("head_pack P=1 (transpose back)", lambda: KERNELS.head_pack(x.view(B, H, N, D), 1))):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "GB/s": round(2 * x.numel() * 2 / ms / 1e6, 1)}))
