# paired-query-block K4: parity, then A/B against the single kernel, then the short bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attn_pair.py -q -x --timeout 120 > gpurun_out/pytest_pair.log 2>&1; echo pair_rc=$?
tail -5 gpurun_out/pytest_pair.log
timeout 300 python -m pytest tests -m gpu -q -x --timeout 300 -k "attention" > gpurun_out/pytest_attn.log 2>&1; echo attn_rc=$?
tail -3 gpurun_out/pytest_attn.log
for rep in 1 2; do for kk in single pair; do MOD_ATTN_KERNEL=$kk timeout 100 python scripts/attn_micro.py 2>&1 | grep '^{' | sed "s/^/$kk /"; done; done
MOD_ATTN_KERNEL=pair timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bench_pair.log 2>&1; echo bench_rc=$?
MOD_ATTN_KERNEL=single timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bench_single.log 2>&1; echo bench_rc=$?
python - <<'PY'
import json
for f in ('gpurun_out/bench_pair.log','gpurun_out/bench_single.log'):
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); print(f, {k:d[k] for k in ('value','attn_ms','attn_tflops','attn_pct_bf16_peak','clocks')})
PY
