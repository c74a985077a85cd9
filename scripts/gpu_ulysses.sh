mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ulysses.py -q -x --timeout 120 > gpurun_out/pytest_uly.log 2>&1; echo uly_rc=$?; tail -3 gpurun_out/pytest_uly.log
timeout 300 python bench.py --ulysses --steps 5 --warmup 3 --no-dense --no-cpu > gpurun_out/bench_uly.log 2>&1; echo bench_rc=$?
python - <<PY
import json
for l in open('gpurun_out/bench_uly.log'):
    if l.startswith('{'):
        d=json.loads(l); print({k:d[k] for k in ('value','ms_per_step','attn_ms','attn_tflops','e2e')}, d['config']['parallelism'])
    elif 'rror' in l: print(l[:300])
PY
python scripts/relayout_time.py 2>&1 | grep '^{' | tee gpurun_out/relayout_time.jsonl
