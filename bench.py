#!/usr/bin/env python
"""bench.py -- MOD-DiT hot path on B200: block-sparse attention fwd (ms, TFLOPS, % of bf16 peak) vs dense
at the HunyuanVideo 720p shape (BASELINE.json "metric", configs[3]).

One STEP = one pass of the whole hot path of SURVEY.md 8(a) at a re-estimation step t_p of
Algorithm 1, on synthetic Family-S inputs resident in HBM:
    K2b mod_predict_block_mask   (Eq. 6/7 + Top-K + CSR)        -> mask for step t
    K4  mod_block_sparse_attn_fwd (Eq. 1 over the index lists)   -> O, lse
    K1  mod_collect_block_stats  (pooled block statistic)       -> fresh W
    K3  mod_update_online_mask   (Eq. 5 + refit (K2a) + roll)
The warm-up (two pooled statistics + fits, keep decision) runs once before timing; K is bisected
so that the mean block sparsity hits --sparsity (default 0.878, the paper's HunyuanVideo
sparsity, Table 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config hunyuan]
Multi-GPU (torchrun): heads are partitioned across ranks (no data-path collective; head-parallel,
SURVEY 8(e)); value = all ranks' attention FLOPs / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic as syn  # noqa: E402

M_WARMUP, DT, T_TOTAL = 12, 10, 50          # Alg. 1 defaults: m = 12, Delta t = 10, T = 50
METRIC = "block-sparse attn fwd ms & TFLOPS (% bf16 peak) vs dense at HunyuanVideo shape"


def attn_flops(row_ptr: np.ndarray, col_idx: np.ndarray, N: int, block: int, D: int) -> float:
    """Algorithmic FLOPs of K4: 4 * D * sum over selected (i,j) of |I_i| * |I_j| (QK^T + PV)."""
    n = row_ptr.shape[-1] - 1
    sizes = np.minimum((np.arange(n) + 1) * block, N) - np.arange(n) * block
    tot = 0
    for rp, ci in zip(row_ptr.reshape(-1, n + 1), col_idx.reshape(-1, col_idx.shape[-1])):
        nnz = rp[-1]
        rows = np.repeat(np.arange(n), np.diff(rp))
        tot += int(np.dot(sizes[rows], sizes[ci[:nnz]]))
    return 4.0 * D * tot


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons}


# ---------------------------------------------------------------------------------------- distributed
# MOD_BENCH_DIST_BACKEND=gloo (bring-up only): run the N>1 code path with gloo for the scalar
# reductions, several ranks sharing the visible GPUs -- validates the multi-rank logic on a 1-GPU box
# (the timings of such a run mean nothing).  The default, and every measured run, is NCCL.
DIST_BACKEND = os.environ.get("MOD_BENCH_DIST_BACKEND", "nccl")


def dist_setup(n_gpus: int):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        if DIST_BACKEND == "gloo":
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if DIST_BACKEND == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if DIST_BACKEND == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------------------------------- our arm
def bisect_top_k(P, x_prev, x_curr, keep, target_sparsity: float, ws: int):
    """Smallest K whose mean block sparsity (over all ranks' heads) is <= target (reading Z8)."""
    n = P.n
    lo, hi = 1, 3 * n - 1

    def sparsity(K):
        rp, _ = P.predict_block_mask(x_prev, x_curr, M_WARMUP - 1, M_WARMUP, M_WARMUP + DT, keep, top_k=K)
        nnz = sum_over_ranks(float(rp[..., -1].sum().item()), ws)
        return 1.0 - nnz / (total_heads * n * n)

    total_heads = sum_over_ranks(float(P.BH), ws)

    while lo < hi:
        mid = (lo + hi) // 2
        if sparsity(mid) <= target_sparsity:
            hi = mid
        else:
            lo = mid + 1
    return lo, sparsity(lo)


def dense_reference_ms(q, k, v, reps: int = 3):
    """Fastest dense attention available on the box (library comparators; context only)."""
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel
    res = {}
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel(be):
                F.scaled_dot_product_attention(q, k, v)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    F.scaled_dot_product_attention(q, k, v)
                e1.record()
                torch.cuda.synchronize()
                res[name] = e0.elapsed_time(e1) / reps
        except Exception as ex:  # backend unavailable for this shape
            res[name] = None
            res[name + "_error"] = str(ex)[:120]
    return res


def run_ours(args):
    import paper_2601_11641_b200 as mod
    from paper_2601_11641_b200 import Plan

    ws, rank, local = dist_setup(args.gpus)
    w_full = syn.CONFIGS[args.config]
    H = w_full.heads
    from paper_2601_11641_b200.parallel import head_range, lpt_head_assignment, ulysses_chunk_heads
    chunks_u = 0
    if args.ulysses:
        # config 5: activations arrive sequence-sharded [B, N/P, H, D]; UlyssesChunkPipeline exchanges head
        # chunks (NCCL all_to_all_single over NVLink) overlapped with the hot path of the previous chunk
        want = args.ulysses_chunks if args.ulysses_chunks > 0 else 3
        chunks_u = max(c for c in range(1, want + 1) if H % (c * ws) == 0)
        heads = ulysses_chunk_heads(H, ws, chunks_u, rank)
    else:
        heads = list(range(*head_range(H, ws, rank)))
    D, N, blk = w_full.head_dim, w_full.tokens, w_full.block
    burst, sustained, hbm, peak_src = load_peaks()

    exact = args.stat == "exact"
    plan_kw = dict(top_k=1, tau_e=0.0, masked_renorm=not exact, attn_kernel=args.attn_kernel)
    extra = {}

    def gen(step):   # this rank's heads of the step's Q, K, V (the bytes one GPU would draw for them)
        if heads == list(range(heads[0], heads[0] + len(heads))):
            return syn.family_s(w_full.with_heads(len(heads)), step=step, seed=syn.SEED_BASE, device="cuda",
                                head_offset=heads[0], total_heads=H)
        return syn.family_s_heads(w_full, heads, step=step, seed=syn.SEED_BASE, device="cuda")

    def warm_stat(P, qq, kk, vv):
        """Statistic of a warm-up step: POOLED, or EXACT Eq. 2 from the dense attention's lse."""
        if not exact:
            return P.collect_block_stats(qq, kk)
        rpd, cid = P.dense_mask()
        _, lsed = P.block_sparse_attn_fwd(qq, kk, vv, rpd, cid)
        torch.cuda.synchronize()
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record()
        U = P.collect_exact_sparsity(qq, kk, lsed, rpd, cid, args.eta)
        e_b.record()
        torch.cuda.synchronize()
        extra["exact_dense_stat_ms"] = round(e_a.elapsed_time(e_b), 3)
        return U

    def warm_up():
        """Warm-up phase of Alg. 1 for this rank's heads: statistics at t = m-1 and t = m,
        fits, keep decision, history (untimed setup)."""
        P_ = Plan(w_full.with_heads(len(heads)), **plan_kw)
        q1, k1, v1 = gen(M_WARMUP - 1)
        W1_ = warm_stat(P_, q1, k1, v1)
        del q1, k1, v1
        q_, k_, v_ = gen(M_WARMUP)
        W2_ = warm_stat(P_, q_, k_, v_)
        xp, xc = P_.fit_mixture(W1_), P_.fit_mixture(W2_)
        return P_, q_, k_, v_, W2_, xp, xc, P_.keep_frames(xp, xc)

    P, q, k, v, W2, x_prev0, x_curr0, keep = warm_up()
    K, sp = bisect_top_k(P, x_prev0, x_curr0, keep, args.sparsity, ws)
    t_step = M_WARMUP + DT                             # t_p^(1) = 22
    lpt_info = None
    if args.lpt and ws > 1 and not args.ulysses:
        # LPT head assignment by the predicted mask nnz of every head (K4 time is proportional to it): all
        # ranks' per-head nnz are gathered, heads are re-dealt greedily, and each rank redoes its warm-up
        import torch.distributed as dist
        rp0, _ = P.predict_block_mask(x_prev0, x_curr0, M_WARMUP - 1, M_WARMUP, t_step, keep, top_k=K)
        nnz_local = torch.zeros(H, dtype=torch.float64, device="cpu" if DIST_BACKEND == "gloo" else "cuda")
        for i, h in enumerate(heads):
            nnz_local[h] = float(rp0[0, i, -1].item())
        dist.all_reduce(nnz_local, op=dist.ReduceOp.SUM)
        cost = nnz_local.cpu().tolist()
        assign = lpt_head_assignment(cost, ws)
        loads = [sum(cost[h] for h in a) for a in assign]
        even = [sum(cost[h] for h in range(*head_range(H, ws, r))) for r in range(ws)]
        lpt_info = {"max_over_mean_load": round(max(loads) / (sum(loads) / ws), 4),
                    "contiguous_max_over_mean_load": round(max(even) / (sum(even) / ws), 4)}
        heads = assign[rank]
        del P, q, k, v, W2
        P, q, k, v, W2, x_prev0, x_curr0, keep = warm_up()
    Hl = len(heads)
    w = w_full.with_heads(Hl)
    hist = W2.clone()                                  # A_hat^(t_p^(0)) = A^(m)
    xs_prev, xs_curr = x_prev0.clone(), x_curr0.clone()
    rp, ci = P.empty_mask()
    o = torch.empty_like(q)
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device="cuda")
    Wf = P.empty_stats()
    stream = torch.cuda.current_stream()
    ev = {k_: [] for k_ in ("attn", "rest")}

    q8 = args.precision == "q8"
    if q8 and exact:
        raise SystemExit("--precision q8 with --stat exact is not supported (the exact statistic needs the bf16 lse)")
    if args.ulysses and (q8 or exact):
        raise SystemExit("--ulysses runs the bf16 pooled step")
    qbuf = P.quant_buffer() if q8 else None

    upipe = None
    if args.ulysses:
        from paper_2601_11641_b200.parallel import UlyssesChunkPipeline
        Ns = N // ws
        qs, ks, vs = syn.family_s_seq_shard(w_full, rank * Ns, (rank + 1) * Ns, step=M_WARMUP, seed=syn.SEED_BASE,
                                            device="cuda")
        o_seq = torch.empty_like(qs)
        upipe = UlyssesChunkPipeline(w_full, chunks_u, **plan_kw)
        assert [h for c in range(chunks_u) for h in upipe.heads(c)] == heads
        hlc = upipe.hl
        uev = []

        def chunk_step(plan, c, qc, kc, vc, oc):
            sl = slice(c * hlc, (c + 1) * hlc)
            st_ = torch.cuda.current_stream()
            e_ = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e_[0].record(st_)
            plan.predict_block_mask(x_prev0[:, sl], x_curr0[:, sl], M_WARMUP - 1, M_WARMUP, t_step, keep[:, sl],
                                    top_k=K, out=(rp[:, sl], ci[:, sl]))
            e_[1].record(st_)
            plan.block_sparse_attn_fwd(qc, kc, vc, rp[:, sl], ci[:, sl], out=oc, lse=lse[:, sl])
            e_[2].record(st_)
            plan.collect_block_stats(qc, kc, out=Wf[:, sl])
            plan.update_online_mask(Wf[:, sl], rp[:, sl], ci[:, sl], hist[:, sl], xs_prev[:, sl], xs_curr[:, sl])
            e_[3].record(st_)
            uev.append(e_)

    overlap_k1 = not (exact or q8 or args.serial_k1)
    side = torch.cuda.Stream() if overlap_k1 else None

    def step(timed_kernels=False):
        if upipe is not None:
            uev.clear()
            upipe.run(qs, ks, vs, o_seq, chunk_step)
            if timed_kernels:
                ev["ulysses"] = ev.get("ulysses", []) + [list(uev)]
            return
        if timed_kernels:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
        P.predict_block_mask(x_prev0, x_curr0, M_WARMUP - 1, M_WARMUP, t_step, keep, top_k=K, out=(rp, ci))
        if timed_kernels:
            e[1].record(stream)
        if overlap_k1:   # K1 reads only Q, K: on a side stream beside K4; K3 joins both below
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                P.collect_block_stats(q, k, out=Wf)
        if q8:   # SURVEY f2 (reading Z30): quantize Q, K, V, then INT8 QK^T / FP8 PV attention
            P.quantize_qkv(q, k, v, out=qbuf)
            P.block_sparse_attn_fwd_q8(qbuf, rp, ci, out=o, lse=lse)
        else:
            P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
        if timed_kernels:
            e[2].record(stream)
        if exact:   # Eq. 2 on the masked map of this step (lse over the kept blocks, reading Z12)
            P.collect_exact_sparsity(q, k, lse, rp, ci, args.eta, out=Wf)
        elif overlap_k1:
            stream.wait_stream(side)
        else:
            P.collect_block_stats(q, k, out=Wf)
        P.update_online_mask(Wf, rp, ci, hist, xs_prev, xs_curr)
        if timed_kernels:
            e[3].record(stream)
            ev["attn"].append((e[1], e[2]))
            ev["rest"].append((e[0], e[1], e[2], e[3]))

    launches_per_step = 3 + (4 if q8 else 1) + (1 if exact else 4) + 6   # predict (3) + attn (+3 quantize) + statistic (pool, split, 2 score passes) + update (6)
    if upipe is not None:   # per chunk: the step + 3 packs / unpacks in, 1 pack + 1 unpack out
        launches_per_step = chunks_u * (launches_per_step + 6 + 2)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rpn, cin = rp.cpu().numpy(), ci.cpu().numpy()
    flops_local = attn_flops(rpn, cin, N, blk, D)
    flops_all = sum_over_ranks(flops_local, ws)
    nnz_local = float(rpn[..., -1].sum())

    # ---- timed region: K steps, barrier + sync on both sides, CUDA events, max over ranks
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(timed_kernels=True)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local, ws)
    if upipe is not None:   # per step: sum over the chunks' events
        attn_ms = statistics.mean(sum(e_[1].elapsed_time(e_[2]) for e_ in st_) for st_ in ev["ulysses"])
        pred_ms = statistics.mean(sum(e_[0].elapsed_time(e_[1]) for e_ in st_) for st_ in ev["ulysses"])
        upd_ms = statistics.mean(sum(e_[2].elapsed_time(e_[3]) for e_ in st_) for st_ in ev["ulysses"])
    else:
        attn_ms = statistics.mean(a.elapsed_time(b) for a, b in ev["attn"])
        pred_ms = statistics.mean(a.elapsed_time(b) for a, b, _, _ in ev["rest"])
        upd_ms = statistics.mean(c.elapsed_time(d) for _, _, c, d in ev["rest"])
    attn_ms_max = max_over_ranks(attn_ms, ws)
    value = flops_all / (ms * 1e-3) / 1e12
    attn_tflops = flops_local / (attn_ms * 1e-3) / 1e12

    out = {"metric": METRIC, "value": round(value, 2), "unit": "TFLOPS", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "int8/e4m3 (f32 softmax)" if q8 else "bf16",
           "data": "synthetic (Family S, seeded; SURVEY 8(d))"}

    # ---- dense comparators (rank 0, 1 GPU shape of its heads): library SDPA + our K4 with all-ones CSR
    dense = {}
    if rank == 0 and not args.no_dense:
        dense = dense_reference_ms(q, k, v)
        rpd, cid = P.dense_mask()
        P.block_sparse_attn_fwd(q, k, v, rpd, cid, out=o, lse=lse)
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        for _ in range(2):
            P.block_sparse_attn_fwd(q, k, v, rpd, cid, out=o, lse=lse)
        d1.record()
        torch.cuda.synchronize()
        dense["ours_all_ones_csr"] = d0.elapsed_time(d1) / 2
        del rpd, cid
    dense_flops = 4.0 * D * N * N * w.batch * w.heads
    fastest = min([x for kk, x in dense.items() if isinstance(x, float)], default=None)

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region.
    # Default path: HeadChunkPipeline overlaps the upload of head chunk c+1, the hot path on chunk c and
    # the download of chunk c-1 on three streams (every step is per head); the q8 / exact /
    # Ulysses variants run serially (upload, step, download on one stream).
    e2e = None
    if not args.no_e2e:
        src = (qs, ks, vs) if upipe is not None else (q, k, v)
        hq, hk, hv = (t.cpu().pin_memory() for t in src)
        ho = torch.empty_like(hq).pin_memory()
        pipelined = not (q8 or exact or upipe is not None) and w.batch == 1
        if pipelined:
            from paper_2601_11641_b200.pipeline import HeadChunkPipeline
            want = args.e2e_chunks
            if want <= 0:   # auto: ~80 MB of upload per chunk (24 chunks at Hunyuan 720p, 4 at CogVideoX)
                want = max(1, round(3 * q.numel() * 2 / (80 << 20)))
            chunks = max(c for c in range(1, min(want, Hl) + 1) if Hl % c == 0)
            pipe = HeadChunkPipeline(w, chunks, top_k=1, tau_e=0.0, masked_renorm=True, attn_kernel=args.attn_kernel)

            def chunk_step(plan, c, qc, kc, vc, oc):
                hs = pipe.heads(c)
                rpc, cic = rp[:, hs], ci[:, hs]
                plan.predict_block_mask(x_prev0[:, hs], x_curr0[:, hs], M_WARMUP - 1, M_WARMUP, t_step, keep[:, hs],
                                        top_k=K, out=(rpc, cic))
                plan.block_sparse_attn_fwd(qc, kc, vc, rpc, cic, out=oc, lse=lse[:, hs])
                plan.collect_block_stats(qc, kc, out=Wf[:, hs])
                plan.update_online_mask(Wf[:, hs], rpc, cic, hist[:, hs], xs_prev[:, hs], xs_curr[:, hs])

            pipe.run(hq, hk, hv, ho, chunk_step)        # untimed warm-up of the pipeline
            torch.cuda.synchronize()
        barrier(ws)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            if pipelined:
                pipe.run(hq, hk, hv, ho, chunk_step)
            elif upipe is not None:
                qs.copy_(hq, non_blocking=True)
                ks.copy_(hk, non_blocking=True)
                vs.copy_(hv, non_blocking=True)
                step()
                ho.copy_(o_seq, non_blocking=True)
            else:
                q.copy_(hq, non_blocking=True)
                k.copy_(hk, non_blocking=True)
                v.copy_(hv, non_blocking=True)
                step()
                ho.copy_(o, non_blocking=True)
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(s0.elapsed_time(s1) / args.steps, ws)
        e2e = {"value": round(flops_all / (e2e_ms * 1e-3) / 1e12, 2), "unit": "TFLOPS",
               "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(3 * q.numel() * 2 * ws),
               "d2h_bytes_per_step": int(o.numel() * 2 * ws),
               "pipeline": (f"{chunks} head chunks on 3 streams (upload / hot path / download overlapped)"
                            if pipelined else "serial (upload, step, download on one stream)")}
        if pipelined:
            del pipe
        del hq, hk, hv, ho

    # ---- roofline of the dominant kernel (K4): algorithmic FLOPs / event-timed launch duration
    # traffic: DRAM bytes per launch from the committed ncu --set full capture of this kernel on this
    # config (profiles/k4_traffic.json), scaled to this rank's heads (each head's bytes are independent)
    traffic, traffic_src = None, None
    kname = P.attn_kernel_name()
    tp = os.path.join(ROOT, "profiles", "k4_traffic.json")
    if os.path.exists(tp):
        try:
            rec = json.load(open(tp)).get(args.config)
            if rec and rec.get("kernel") == kname:
                traffic = round(rec["bytes"] * Hl / rec["heads"])
                traffic_src = f"{rec['source']}; x {Hl}/{rec['heads']} heads"
        except Exception:
            traffic = None
    # the quantized kernel's peak: the measured bf16 figure x the guide's nominal 2x ratio for 8-bit MMAs
    pk = burst * (2 if q8 else 1)
    roof = {"bound": "tensor", "achieved": round(attn_tflops, 1), "peak": pk, "unit": "TFLOP/s",
            "frac": round(attn_tflops / pk, 4), "frac_of_sustained": round(attn_tflops / (sustained * (2 if q8 else 1)), 4),
            "peak_source": peak_src + (" (bf16 x 2, nominal 8-bit ratio)" if q8 else ""),
            "traffic": None if q8 else traffic, "traffic_source": None if q8 else traffic_src,
            "kernel": "quantize (3 kernels) + attn_q8_kernel" if q8 else kname,
            "algorithmic_flops_per_launch": flops_local}

    out.update({
        "config": {"workload": f"{w_full.name}: B={w_full.batch} H={w_full.heads} D={D} N={N} "
                               f"({w_full.frames}x{w_full.height}x{w_full.width}+{w_full.prefix_tokens}), block {blk}",
                   "heads_per_rank": Hl, "top_k": K, "block_sparsity": round(sp, 4),
                   "target_sparsity": args.sparsity, "nnz_blocks_rank0": nnz_local,
                   "step": ("predict(K2b) + attn(K4) + stats(K1) + update(K3: Eq.5 + fit K2a + roll) at t_p=22"
                            + (" (K1 on a side stream beside K4)" if overlap_k1 else "")),
                   "l2": "inputs larger than L2 (Q,K,V = %.2f GB per rank > 126 MB)" % (3 * q.numel() * 2 / 1e9),
                   "parallelism": (f"ulysses a2a in {chunks_u} overlapped head chunks + head-parallel x{ws}"
                                   if args.ulysses else
                                   (f"head-parallel x{ws} (LPT by mask nnz)" if lpt_info else f"head-parallel x{ws}")),
                   **({"lpt": lpt_info} if lpt_info else {})},
        "attn_ms": round(attn_ms_max, 3), "attn_tflops": round(attn_tflops, 1),
        "attn_pct_bf16_peak": round(100 * attn_tflops / burst, 1),
        "pipeline_overhead_ms": {"predict": round(pred_ms, 4), "stats_update": round(upd_ms, 4)},
        "dense_ms": {kk: (round(x, 3) if isinstance(x, float) else x) for kk, x in dense.items()},
        "dense_tflops_fastest": round(dense_flops / (fastest * 1e-3) / 1e12, 1) if fastest else None,
        "speedup_vs_fastest_dense": round(fastest / attn_ms, 3) if fastest else None,
        "roofline": roof, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(), "library": mod.LIB_PATH, "statistic": args.stat, **extra,
    })

    # ---- cpu baseline: the oracle as it stands on a bounded sample (rank 0, N=1 only)
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(w, q, k, v, rpn, cin, args.cpu_seconds, x_prev0, x_curr0, keep, K)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(w, q, k, v, rpn, cin, budget_s: float, x_prev0=None, x_curr0=None, keep=None, K=None, Wf=None):
    """The oracle as it stands, timed on the host cores, rank 0 at N = 1:
    * the mask pipeline of one head at full n^2 scale, timed in full: pooled statistic (O2), fit (O4,
      Cholesky of the p x p Gram), predict + select + mask (O6-O8) and the Eq. 5 update + refit (O10);
    * masked attention (O9) on sampled query blocks of head 0 under the bench's own mask (its TFLOPS is
      the line's ``value``), and the full-shape attention time EXTRAPOLATED from the sample by the
      selected-block count of all heads."""
    import oracle as O
    L = O.make_layout(1, 1, w.head_dim, w.prefix_tokens, w.frames, w.height, w.width, w.block)
    mask = O.csr_to_mask(rpn[0, 0], cin[0, 0], L.n)
    qh, kh, vh = (t[:, :1].cpu() for t in (q, k, v))
    pipe = {}
    t0 = time.perf_counter()
    W = O.pooled_block_stats(qh, kh, L)
    pipe["stats_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    X = O.fit_mixture(W, L)
    pipe["fit_s"] = time.perf_counter() - t0
    if x_prev0 is not None:
        xp = x_prev0[:, :1].double().cpu().numpy()
        xc = x_curr0[:, :1].double().cpu().numpy()
        kp = keep[:, :1].cpu().numpy()
        t0 = time.perf_counter()
        O.predict_block_mask(xp, xc, M_WARMUP - 1, M_WARMUP, M_WARMUP + DT, kp, L, O.SELECT_TOPK, K)
        pipe["predict_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        hist = O.reconstruct_history(W, W.copy(), mask[None, None], True)
        O.fit_mixture(hist, L)
        pipe["update_s"] = time.perf_counter() - t0
    del X
    rng = np.random.default_rng(0)
    order = rng.permutation(L.n)
    t0 = time.perf_counter()
    flops, nb, blocks_done = 0.0, 0, 0
    for i in order:
        O.masked_attention_rows(qh, kh, vh, mask, L, 0, 0, [int(i)])
        lo, hi = L.block_range(int(i))
        keys = sum(L.block_size(j) for j in np.nonzero(mask[i])[0])
        flops += 4.0 * w.head_dim * (hi - lo) * keys
        blocks_done += int(mask[i].sum())
        nb += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    total_blocks = float(rpn[..., -1].sum())
    return {"value": flops / dt / 1e12, "unit": "TFLOPS", "cores": os.cpu_count(), "kind": "oracle",
            "cpu_model": _cpu_model(), "threads": torch.get_num_threads(),
            "sample": f"{nb} query blocks of head 0 (oracle masked_attention_rows, fp64 numpy, the bench's mask), "
                      f"{dt:.1f} s; mask pipeline of head 0 at full n^2 scale timed in full",
            "pipeline_one_head_s": {k_: round(v_, 3) for k_, v_ in pipe.items()},
            "attention_full_shape_s_extrapolated": round(dt / max(blocks_done, 1) * total_blocks, 1),
            "extrapolation": "sampled seconds per selected block x selected blocks of all heads (labelled, not run)"}


# ---------------------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle timed on the host cores (the 'reference' of this tier), bounded sample per step."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    w = syn.CONFIGS[args.config].with_heads(1)
    L = O.make_layout(1, 1, w.head_dim, w.prefix_tokens, w.frames, w.height, w.width, w.block)
    gen = dict(seed=syn.SEED_BASE, device="cpu", total_heads=syn.CONFIGS[args.config].heads)
    q1, k1, _ = syn.family_s(w, step=M_WARMUP - 1, **gen)
    q, k, v = syn.family_s(w, step=M_WARMUP, **gen)
    W1 = O.pooled_block_stats(q1, k1, L)
    W2 = O.pooled_block_stats(q, k, L)
    x1, x2 = O.fit_mixture(W1, L), O.fit_mixture(W2, L)
    keep = O.keep_frames(x1, x2, L, 0.0)
    n = L.n
    lo, hi = 1, 3 * n - 1
    while lo < hi:                                     # same K rule as our arm, evaluated by the oracle
        mid = (lo + hi) // 2
        m_ = O.predict_block_mask(x1, x2, M_WARMUP - 1, M_WARMUP, M_WARMUP + DT, keep, L, O.SELECT_TOPK, mid)
        if 1.0 - m_.mean() <= args.sparsity:
            hi = mid
        else:
            lo = mid + 1
    K = lo
    rng = np.random.default_rng(0)
    sample_blocks = int(args.ref_blocks)

    def step():
        masks = O.predict_block_mask(x1, x2, M_WARMUP - 1, M_WARMUP, M_WARMUP + DT, keep, L, O.SELECT_TOPK, K)
        blocks = rng.choice(n, size=sample_blocks, replace=False)
        O.masked_attention_rows(q, k, v, masks[0, 0], L, 0, 0, [int(b) for b in blocks])
        fl = sum(4.0 * w.head_dim * L.block_size(int(i)) * sum(L.block_size(j) for j in np.nonzero(masks[0, 0, i])[0])
                 for i in blocks)
        return fl

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    fl = 0.0
    for _ in range(args.steps):
        fl += step()
    dt = time.perf_counter() - t0
    val = fl / dt / 1e12
    out = {"metric": METRIC, "value": val, "unit": "TFLOPS", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (Family S, seeded)", "impl": "reference",
           "config": {"workload": f"{syn.CONFIGS[args.config].name} (oracle sample: head 0, {sample_blocks} query "
                                  f"blocks per step)", "top_k": K},
           "cpu_baseline": {"value": val, "unit": "TFLOPS", "cores": os.cpu_count(), "kind": "oracle",
                            "sample": f"{sample_blocks} random query blocks of head 0 per step"},
           "e2e": {"value": val, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _self_launch(n: int) -> None:
    """`python bench.py --gpus N` without a launcher: re-exec under torch.distributed.run with N ranks
    (one process per GPU, rendezvous on 127.0.0.1) and exit with its status."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="hunyuanvideo-720p", choices=sorted(syn.CONFIGS))
    ap.add_argument("--sparsity", type=float, default=0.878)
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--serial-k1", action="store_true",
                    help="run K1 after K4 on one stream (default: K1 on a side stream beside K4, K3 joins both)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="head chunks of the pipelined e2e leg (0: about 80 MB of upload per chunk)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-blocks", type=int, default=4)
    ap.add_argument("--precision", default="bf16", choices=["bf16", "q8"],
                    help="attention operands: bf16 (headline) or the Sage-style INT8/FP8 path (SURVEY f2)")
    ap.add_argument("--stat", default="pooled", choices=["pooled", "exact"],
                    help="block statistic: pooled (north_star (1)) or the paper's exact Eq. 2 (SURVEY f1)")
    ap.add_argument("--eta", type=float, default=1e-4)
    ap.add_argument("--attn-kernel", default="default", choices=["default", "splitkv", "pair", "wide"],
                    help="K4 schedule (include/moddit.h mod_attn_kernel); default is the headline kernel")
    ap.add_argument("--ulysses", action="store_true",
                    help="sequence-sharded inputs: Ulysses all-to-all in and out of every step (config 5)")
    ap.add_argument("--ulysses-chunks", type=int, default=0,
                    help="head chunks of the overlapped Ulysses exchange (0: up to 3 that divide H / P)")
    ap.add_argument("--lpt", action="store_true",
                    help="head-parallel: deal heads to ranks by longest-processing-time on the predicted mask nnz")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _self_launch(args.gpus)
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws_env}: launch one rank per GPU")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
