"""CPU baseline coverage of BASELINE.md §3: the fp64 oracle (as it stands, test infrastructure) timed on this
box's host cores for the FULL Alg.-1 re-estimation step -- warm-up statistics and fits, keep, predict,
full masked attention over every head, fresh statistic, Eq. 5 update + refit -- on the tiny and the
CogVideoX-5B shapes (Family S, the same seeded bytes the GPU path reads), one JSON line per config with
the CPU model, core and thread counts.  Hunyuan / Wan are covered by bench.py's cpu_baseline (full n^2
pipeline of one head, sampled attention, extrapolated full-shape attention, labelled as such).
  python scripts/cpu_baseline_configs.py [--configs tiny,cogvideox-5b]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synthetic as syn  # noqa: E402
from bench import _cpu_model  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="tiny,cogvideox-5b")
    ap.add_argument("--sparsity", type=float, default=0.878)
    args = ap.parse_args()
    for name in args.configs.split(","):
        w = syn.CONFIGS[name]
        L = O.make_layout(w.batch, w.heads, w.head_dim, w.prefix_tokens, w.frames, w.height, w.width, w.block)
        t = {}
        q1, k1, _ = syn.family_s(w, step=11)
        q, k, v = syn.family_s(w, step=12)
        T0 = time.perf_counter()
        W1 = O.pooled_block_stats(q1, k1, L)
        W2 = O.pooled_block_stats(q, k, L)
        t["stats_x2_s"] = time.perf_counter() - T0
        T0 = time.perf_counter()
        x1, x2 = O.fit_mixture(W1, L), O.fit_mixture(W2, L)
        t["fit_x2_s"] = time.perf_counter() - T0
        keep = O.keep_frames(x1, x2, L)
        # K for the target sparsity on the oracle's own prediction (bisection; untimed)
        lo_, hi_ = 1, 3 * L.n - 1
        def sp(K):
            m = O.predict_block_mask(x1, x2, 11, 12, 22, keep, L, top_k=K)
            return 1.0 - m.sum() / m.size
        while lo_ < hi_:
            mid = (lo_ + hi_) // 2
            if sp(mid) <= args.sparsity:
                hi_ = mid
            else:
                lo_ = mid + 1
        K = lo_
        T0 = time.perf_counter()
        masks = O.predict_block_mask(x1, x2, 11, 12, 22, keep, L, top_k=K)
        t["predict_s"] = time.perf_counter() - T0
        T0 = time.perf_counter()
        o, lse = O.masked_attention(q, k, v, masks, L)
        t["attention_s"] = time.perf_counter() - T0
        T0 = time.perf_counter()
        Wf = O.pooled_block_stats(q, k, L)
        t["stats_s"] = time.perf_counter() - T0
        T0 = time.perf_counter()
        O.update_online_mask(Wf, W2.copy(), masks, x1, x2, L)
        t["update_s"] = time.perf_counter() - T0
        # selected-block FLOPs of the attention (4 D |I_i| |I_j| per block)
        sizes = np.array([L.block_size(i) for i in range(L.n)], dtype=np.float64)
        flops = float(4 * w.head_dim * np.einsum("bhij,i,j->", masks.astype(np.float64), sizes, sizes))
        step_s = t["predict_s"] + t["attention_s"] + t["stats_s"] + t["update_s"]
        print(json.dumps({"config": name, "kind": "oracle (fp64 numpy), full re-estimation step, not extrapolated",
                          "cpu_model": _cpu_model(), "cores": os.cpu_count(), "threads": torch.get_num_threads(),
                          "top_k": K, "block_sparsity": round(float(1.0 - masks.mean()), 4),
                          "attention_tflop": round(flops / 1e12, 4),
                          "attention_tflops": round(flops / t["attention_s"] / 1e12, 6),
                          "step_s": round(step_s, 3), **{k_: round(v_, 3) for k_, v_ in t.items()}}), flush=True)


if __name__ == "__main__":
    main()
