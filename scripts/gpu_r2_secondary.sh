# round-2 secondary measurements: sparsity sweep / interval / T=50 run (with and without drift), analysis
# metrics (with drift), BASELINE configs 2-3 bench lines, plan creation times
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python scripts/sweep_interval.py > gpurun_out/sweep_interval_hunyuan.jsonl 2> gpurun_out/sweep.err; tail -2 gpurun_out/sweep.err; wc -l gpurun_out/sweep_interval_hunyuan.jsonl
timeout 900 python scripts/sweep_interval.py --parts interval,run --drift 1.0 > gpurun_out/sweep_interval_hunyuan_drift.jsonl 2> gpurun_out/sweep_d.err; tail -2 gpurun_out/sweep_d.err
timeout 900 python scripts/analysis_metrics.py --drift 1.0 > gpurun_out/analysis_hunyuan_drift.jsonl 2> gpurun_out/an.err; tail -2 gpurun_out/an.err
for c in cogvideox-5b wan2.1-14b-720p; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e >> gpurun_out/bench_configs.jsonl 2> gpurun_out/bc_$c.err || tail -3 gpurun_out/bc_$c.err; done
python - <<'PY' > gpurun_out/plan_create_ms.jsonl
import json, torch, synthetic as syn
from paper_2601_11641_b200 import Plan
for name in ("tiny", "cogvideox-5b", "wan2.1-14b-720p", "hunyuanvideo-720p"):
    w = syn.CONFIGS[name]
    P = Plan(w)
    print(json.dumps({"config": name, "n": P.n, "p": P.p, "plan_create_ms": round(P.create_ms, 1), "solver": P.solver,
                      "min_pivot": P.min_pivot, "null_dim": P.null_dim}))
PY
cat gpurun_out/plan_create_ms.jsonl
