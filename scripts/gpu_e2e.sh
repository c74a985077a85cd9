mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x --timeout 120 > gpurun_out/pytest_pipe.log 2>&1; echo pipe_rc=$?; tail -3 gpurun_out/pytest_pipe.log
for c in 8 4; do timeout 400 python bench.py --steps 5 --warmup 3 --no-dense --no-cpu --e2e-chunks $c > gpurun_out/bench_e2e_$c.log 2>&1; echo bench_rc=$?
python - <<PY
import json
for l in open('gpurun_out/bench_e2e_$c.log'):
    if l.startswith('{'):
        d=json.loads(l); print($c, {k:d[k] for k in ('value','ms_per_step','attn_tflops','e2e','clocks')})
    elif 'Error' in l or 'error' in l: print(l[:300])
PY
done
