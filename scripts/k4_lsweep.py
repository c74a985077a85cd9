"""K4 time against the list length L (every row lists L random blocks incl. its diagonal) at a config's
shape: separates the per-item (per query block) cost from the per-block cost of each schedule.
  python scripts/k4_lsweep.py [config] [kernels,comma-separated] [L values,comma-separated]
Prints one JSON line per (kernel, L): ms, ns per item, cycles per block at the measured SM clock."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import threading
import time

import torch

import synthetic as syn
import paper_2601_11641_b200 as M

# EXTRA_KERNELS="name=enum,...": schedules of a variant library (MODDIT_LIB_OVERRIDE) the binding does not name
for spec in filter(None, os.environ.get("EXTRA_KERNELS", "").split(",")):
    from paper_2601_11641_b200 import _lib
    _lib.ATTN_KERNELS.setdefault(spec.split("=")[0], int(spec.split("=")[1]))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cogvideox-5b"
kerns = (sys.argv[2] if len(sys.argv) > 2 else "default,wide").split(",")
Ls = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "2,4,8,17,32,64").split(",")]
w = syn.CONFIGS[cfg]
REPS = int(os.environ.get("REPS", "10"))


class Clocks:
    """SM clock (MHz) and board power (W) sampled by NVML every 2 ms while active."""

    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.mhz, self.w, self.on = [], [], False

    def _run(self):
        while self.on:
            self.mhz.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.w.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            time.sleep(0.002)

    def __enter__(self):
        self.mhz, self.w, self.on = [], [], True
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.on = False
        self.t.join()

    def median(self):
        import statistics
        return (statistics.median(self.mhz) if self.mhz else None, statistics.median(self.w) if self.w else None)


clk = Clocks()
q, k, v = syn.family_r(w, seed=5, device="cuda")
P0 = M.Plan(w)
n = P0.n
BH = w.batch * w.heads
g = torch.Generator(device="cpu").manual_seed(3)
for L in Ls:
    # row i: its diagonal plus L-1 distinct other blocks, ascending
    r = torch.rand(BH, n, n, generator=g)
    idx = torch.arange(n)
    r[:, idx, idx] = -1.0
    sel = torch.topk(-r, L, dim=-1).indices.sort(dim=-1).values.int()
    rp = (torch.arange(n + 1, dtype=torch.int32) * L).repeat(BH, 1).reshape(w.batch, w.heads, n + 1)
    ci = torch.zeros(w.batch, w.heads, n * n, dtype=torch.int32)
    ci[..., : n * L] = sel.reshape(w.batch, w.heads, n * L)
    rp, ci = rp.cuda(), ci.cuda()
    for kern in kerns:
        P = M.Plan(w, attn_kernel=kern)
        o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
        for _ in range(2):
            P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = REPS
        torch.cuda.synchronize()
        with clk:
            e0.record(st)
            for _ in range(reps):
                P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
            e1.record(st)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        mhz, watts = clk.median()
        items_per_sm = BH * n / 148
        print(json.dumps({"config": cfg, "kernel": P.attn_kernel_name(), "L": L, "ms": round(ms, 4),
                          "us_per_item_per_sm": round(ms * 1e3 / items_per_sm, 3),
                          "ns_per_block_per_sm": round(ms * 1e6 / (items_per_sm * L), 1),
                          "sm_mhz": mhz, "watts": watts,
                          "cycles_per_block": round(ms * 1e6 / (items_per_sm * L) * mhz / 1e3, 0) if mhz else None}),
              flush=True)
