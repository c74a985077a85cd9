# quick loop: attention parity + short bench (no dense / e2e / cpu legs)
mkdir -p gpurun_out
timeout 150 python -m pytest tests -m gpu -q -x --timeout 300 -k "attention" > gpurun_out/pytest_attn.log 2>&1; echo attn_rc=$?
tail -3 gpurun_out/pytest_attn.log
timeout 200 python bench.py --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bench_quick.log 2>&1; echo bench_rc=$?
python - <<'PY'
import json
for l in open('gpurun_out/bench_quick.log'):
    if l.startswith('{'):
        d=json.loads(l); print({k:d[k] for k in ('value','ms_per_step','attn_ms','attn_tflops','attn_pct_bf16_peak','pipeline_overhead_ms','clocks')})
    else: print(l.rstrip()[:300])
PY
