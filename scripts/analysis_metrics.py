"""App. A analysis metrics on synthetic Family-S trajectories, computed by the GPU path.

  nae         NAE of the three-pattern fit of the pooled map at t = m, per config (Fig. 4 / P:254-259:
              "NAE vs sequence length");
  der         DER(t) = ||S^(t) - S^(12)|| / ||S^(12)|| for t = 13..50;
  recon       NRE(t_p) of Eq. 5's reconstructed map vs the fresh full map at t_p = 22, 32, 42;
  linearity   NRE of the Eq. 6/7 prediction of every C/D intensity over (22, 32];
  timing      map_rel_error / linearity_nre kernel times vs their HBM floors.
Family S re-draws only the noise per step, so its maps drift little: these runs exercise the metrics
at the real shapes; they do not reproduce the paper's figures (which need the models).
  python scripts/analysis_metrics.py [--config hunyuanvideo-720p]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic as syn  # noqa: E402
from bench import DT, M_WARMUP, T_TOTAL, bisect_top_k, load_peaks  # noqa: E402
from paper_2601_11641_b200 import Plan  # noqa: E402


def summary(x):
    x = np.asarray(x, dtype=np.float64)
    x = x[np.isfinite(x)]
    return {"mean": float(x.mean()), "p50": float(np.median(x)), "max": float(x.max())} if x.size else None


def timed(fn, reps=20):
    """Device time per call: ``reps`` calls captured in one CUDA graph (the launches are a few us of
    GPU work each, so host-side ctypes overhead would otherwise be what the events measure)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hunyuanvideo-720p", choices=sorted(syn.CONFIGS))
    ap.add_argument("--drift", type=float, default=0.0,
                    help="Family S pattern-strength drift over the denoising steps (synthetic/__init__.py)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    gen = dict(seed=syn.SEED_BASE, device="cuda", drift=args.drift)
    _, _, hbm, _ = load_peaks()

    for name in ("tiny", "cogvideox-5b", "wan2.1-14b-720p", "hunyuanvideo-720p"):
        if name not in syn.CONFIGS:
            continue
        w = syn.CONFIGS[name]
        P = Plan(w)
        q, k, _ = syn.family_s(w, step=M_WARMUP, **gen)
        _, nae = P.fit_mixture(P.collect_block_stats(q, k), want_nae=True)
        print(json.dumps({"drift": args.drift, "part": "nae", "config": name, "tokens": w.tokens, "n": P.n, "p": P.p,
                          "nae": summary(nae.double().cpu().numpy())}), flush=True)
        del q, k

    w = syn.CONFIGS[args.config]
    P = Plan(w, top_k=1, masked_renorm=True)
    maps, fits = {}, {}
    for t in range(M_WARMUP - 1, T_TOTAL + 1):
        q, k, _ = syn.family_s(w, step=t, **gen)
        maps[t] = P.collect_block_stats(q, k)
        fits[t] = P.fit_mixture(maps[t])
        del q, k
    der = {t: P.map_rel_error(maps[t], maps[M_WARMUP]).cpu().numpy().ravel() for t in range(M_WARMUP + 1, T_TOTAL + 1)}
    print(json.dumps({"drift": args.drift, "part": "der", "config": args.config,
                      "der_mean_over_heads": {t: round(float(v.mean()), 6) for t, v in der.items()},
                      "der_max": float(max(v.max() for v in der.values()))}), flush=True)

    # Eq. 5 over the schedule's re-estimation steps with the pipeline's own masks
    keep = P.keep_frames(fits[M_WARMUP - 1], fits[M_WARMUP])
    K, sp = bisect_top_k(P, fits[M_WARMUP - 1], fits[M_WARMUP], keep, 0.878, 1)
    hist = maps[M_WARMUP].clone()
    xp, xc = fits[M_WARMUP - 1].clone(), fits[M_WARMUP].clone()
    tprev, tcurr = M_WARMUP - 1, M_WARMUP
    rec = {}
    for tp in range(M_WARMUP + DT, T_TOTAL + 1, DT):
        rp, ci = P.predict_block_mask(xp, xc, tprev, tcurr, tp, keep, top_k=K)
        P.update_online_mask(maps[tp], rp, ci, hist, xp, xc)
        tprev, tcurr = tcurr, tp
        rec[tp] = summary(P.map_rel_error(hist, maps[tp]).cpu().numpy())
    print(json.dumps({"drift": args.drift, "part": "recon", "config": args.config, "top_k": K, "block_sparsity": round(sp, 4),
                      "nre_vs_fresh_full_map": rec}), flush=True)

    # linearity of the true fits over (22, 32] against the Eq. 6 line through X^(12), X^(22)
    ts = list(range(M_WARMUP + DT + 1, M_WARMUP + 2 * DT + 1))
    traj = torch.stack([fits[t] for t in ts]).contiguous()
    nre = P.linearity_nre(fits[M_WARMUP], fits[M_WARMUP + DT], M_WARMUP, M_WARMUP + DT, traj, ts).cpu().numpy()
    fin = nre[np.isfinite(nre)]
    print(json.dumps({"drift": args.drift, "part": "linearity", "config": args.config, "window": [ts[0] - 1, ts[-1]],
                      "patterns": int(nre.size), "nre": summary(nre),
                      "frac_strong_linearity_lt_0.1": round(float((fin < 0.1).mean()), 4) if fin.size else None}),
          flush=True)

    BH, n, p = w.batch * w.heads, P.n, P.p
    P.workspace()
    rel_out = torch.empty((w.batch, w.heads), dtype=torch.float64, device="cuda")
    ms_rel = timed(lambda: P.map_rel_error(maps[T_TOTAL], maps[M_WARMUP], out=rel_out))
    ms_lin = timed(lambda: P.linearity_nre(fits[M_WARMUP], fits[M_WARMUP + DT], M_WARMUP, M_WARMUP + DT, traj, ts))
    b_rel = 2 * BH * n * n * 4
    b_lin = (2 + len(ts)) * BH * p * 8 + BH * (3 * n - 1) * 8
    print(json.dumps({"drift": args.drift, "part": "timing", "config": args.config,
                      "map_rel_error_us": round(ms_rel * 1e3, 1), "map_rel_error_gbs": round(b_rel / ms_rel / 1e6, 1),
                      "map_rel_error_bytes": b_rel,
                      "linearity_nre_us": round(ms_lin * 1e3, 1), "linearity_nre_gbs": round(b_lin / ms_lin / 1e6, 1),
                      "linearity_nre_bytes": b_lin, "hbm_peak_gbs": hbm}), flush=True)


if __name__ == "__main__":
    main()
