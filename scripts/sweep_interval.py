"""Secondary measurements of SURVEY 8(d) at the HunyuanVideo 720p shape on one B200 (BASELINE configs 4-5):

  sweep     K4 at mean block sparsity 50/60/70/80/87.8/90 % (K bisected on the pipeline's own
            prediction, Family-S inputs) vs the fastest dense attention on the box (cuDNN SDPA);
  interval  one denoising interval (22, 32] of Algorithm 1 driven by Schedule: 10 x (K2b + K4)
            plus one re-estimation (K1 + K3 + refit) at t_p = 32 -- the mask pipeline's share of
            the interval is the paper's "1-2 % overhead" claim;
  run       the whole T = 50 schedule of one layer (12 dense warm-up steps, 38 sparse steps) vs 50
            dense steps, i.e. the attention-level analogue of the paper's end-to-end speedup.

Each step's features are Family S at that step (synthetic, seeded); they are generated outside the
timed regions. Times are CUDA events on the current stream. Prints one JSON line per measurement.
  python scripts/sweep_interval.py [--config hunyuanvideo-720p] [--parts sweep,interval,run]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthetic as syn  # noqa: E402
from bench import (DT, M_WARMUP, T_TOTAL, attn_flops, bisect_top_k, dense_reference_ms,  # noqa: E402
                   load_peaks)

import paper_2601_11641_b200 as mod  # noqa: E402,F401
from paper_2601_11641_b200 import Plan  # noqa: E402
from paper_2601_11641_b200.schedule import Schedule  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def time_k4(P, q, k, v, rp, ci, reps=10):
    o, lse = P.block_sparse_attn_fwd(q, k, v, rp, ci)
    for _ in range(2):
        P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record()
        P.block_sparse_attn_fwd(q, k, v, rp, ci, out=o, lse=lse)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts), max(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hunyuanvideo-720p", choices=sorted(syn.CONFIGS))
    ap.add_argument("--drift", type=float, default=0.0,
                    help="Family S pattern-strength drift over the denoising steps (synthetic/__init__.py)")
    ap.add_argument("--parts", default="sweep,interval,run")
    ap.add_argument("--sparsity", type=float, default=0.878, help="target for interval/run")
    args = ap.parse_args()
    parts = set(args.parts.split(","))
    w = syn.CONFIGS[args.config]
    D, N, blk = w.head_dim, w.tokens, w.block
    burst, sustained, _, _ = load_peaks()
    torch.cuda.set_device(0)
    P = Plan(w, top_k=1, tau_e=0.0)
    gen = dict(seed=syn.SEED_BASE, device="cuda", drift=args.drift)

    # warm-up statistics at t = m-1, m (as bench.py) -> fits, keep, K for each target sparsity
    q, k, v = syn.family_s(w, step=M_WARMUP - 1, **gen)
    W1 = P.collect_block_stats(q, k)
    q, k, v = syn.family_s(w, step=M_WARMUP, **gen)
    W2 = P.collect_block_stats(q, k)
    x_prev, x_curr = P.fit_mixture(W1), P.fit_mixture(W2)
    keep = P.keep_frames(x_prev, x_curr)
    dense = dense_reference_ms(q, k, v)
    dense_ms = min(x for key, x in dense.items() if isinstance(x, float))
    dense_flops = 4.0 * D * N * N * w.heads * w.batch

    if "sweep" in parts:
        for target in (0.5, 0.6, 0.7, 0.8, 0.878, 0.9):
            K, sp = bisect_top_k(P, x_prev, x_curr, keep, target, 1)
            rp, ci = P.predict_block_mask(x_prev, x_curr, M_WARMUP - 1, M_WARMUP, M_WARMUP + DT, keep, top_k=K)
            fl = attn_flops(rp.cpu().numpy(), ci.cpu().numpy(), N, blk, D)
            med, lo, hi = time_k4(P, q, k, v, rp, ci)
            print(json.dumps({"drift": args.drift, "part": "sweep", "config": args.config, "target_sparsity": target, "top_k": K,
                              "block_sparsity": round(sp, 4), "tflop": round(fl / 1e12, 3), "k4_ms": round(med, 3),
                              "k4_ms_min": round(lo, 3), "k4_ms_max": round(hi, 3),
                              "tflops": round(fl / med / 1e9, 1), "pct_burst": round(100 * fl / med / 1e9 / burst, 1),
                              "dense_ms": round(dense_ms, 3), "speedup_vs_dense": round(dense_ms / med, 2),
                              "dense_comparators": {kk: (round(x, 3) if isinstance(x, float) else x)
                                                    for kk, x in dense.items() if not kk.endswith("_error")}}),
                  flush=True)

    if "interval" in parts or "run" in parts:
        K, sp = bisect_top_k(P, x_prev, x_curr, keep, args.sparsity, 1)
        S = Schedule(P, T=T_TOTAL, m=M_WARMUP, dt=DT, top_k=K)
        o = torch.empty_like(q)
        lse = torch.empty(q.shape[:-1], dtype=torch.float32, device="cuda")
        per_step, snap = [], None
        for t in range(1, T_TOTAL + 1):
            qt, kt, vt = syn.family_s(w, step=t, **gen)
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record()
            S.step(t, qt, kt, vt, out=o, lse=lse)
            b.record()
            torch.cuda.synchronize()
            per_step.append(a.elapsed_time(b))
            if t == M_WARMUP + DT:   # state entering the interval (22, 32]
                snap = {key: (x.clone() if torch.is_tensor(x) else x) for key, x in vars(S.state).items()}
            del qt, kt, vt
        if "interval" in parts:
            # replay (22, 32] from the snapshot with events around every call (Schedule.step's order)
            st = snap
            calls = {"predict": 0.0, "attn": 0.0, "stats": 0.0, "update": 0.0}
            win = list(range(M_WARMUP + DT + 1, M_WARMUP + 2 * DT + 1))
            for t in win:
                qt, kt, vt = syn.family_s(w, step=t, **gen)
                torch.cuda.synchronize()
                e = [ev() for _ in range(5)]
                e[0].record()
                rp, ci = P.predict_block_mask(st["x_prev"], st["x_curr"], st["t_prev"], st["t_curr"], t, st["keep"],
                                              top_k=K)
                e[1].record()
                _, l = P.block_sparse_attn_fwd(qt, kt, vt, rp, ci, out=o, lse=lse)
                e[2].record()
                upd = S.is_update_step(t)
                if upd:
                    Wt = P.collect_block_stats(qt, kt)
                    e[3].record()
                    P.update_online_mask(Wt, rp, ci, st["hist"], st["x_prev"], st["x_curr"])
                    st["t_prev"], st["t_curr"] = st["t_curr"], t
                    e[4].record()
                torch.cuda.synchronize()
                calls["predict"] += e[0].elapsed_time(e[1])
                calls["attn"] += e[1].elapsed_time(e[2])
                if upd:
                    calls["stats"] += e[2].elapsed_time(e[3])
                    calls["update"] += e[3].elapsed_time(e[4])
                del qt, kt, vt
            tot = sum(calls.values())
            over = tot - calls["attn"]
            print(json.dumps({"drift": args.drift, "part": "interval", "config": args.config, "window": [win[0] - 1, win[-1]],
                              "top_k": K, "block_sparsity": round(sp, 4),
                              "schedule_interval_ms": round(sum(per_step[t - 1] for t in win), 3),
                              "replay_ms": {key: round(x, 3) for key, x in calls.items()},
                              "mask_pipeline_ms": round(over, 3), "mask_pipeline_pct": round(100 * over / tot, 2),
                              "note": "10 x (K2b predict + K4) + 1 x (K1 stats + K3 update/refit) at t_p = 32; "
                                      "schedule_interval_ms is Schedule.step end to end (Python included)"}),
                  flush=True)
        if "run" in parts:
            dense_total = sum(per_step[t - 1] for t in range(1, M_WARMUP + 1))
            sparse_total = sum(per_step[t - 1] for t in range(M_WARMUP + 1, T_TOTAL + 1))
            all_dense = T_TOTAL * dense_ms
            print(json.dumps({"drift": args.drift, "part": "run", "config": args.config, "T": T_TOTAL, "m": M_WARMUP, "dt": DT,
                              "top_k": K, "block_sparsity": round(sp, 4),
                              "warmup_ms": round(dense_total, 1), "sparse_steps_ms": round(sparse_total, 1),
                              "schedule_total_ms": round(dense_total + sparse_total, 1),
                              "all_dense_cudnn_ms": round(all_dense, 1),
                              "speedup_vs_all_dense": round(all_dense / (dense_total + sparse_total), 2),
                              "dense_flops_per_step_tflop": round(dense_flops / 1e12, 2),
                              "note": "warm-up steps run our K4 with the all-ones index list plus the two "
                                      "warm-up statistics/fits; one attention layer"}), flush=True)


if __name__ == "__main__":
    main()
