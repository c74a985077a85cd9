# K4 variant A/B (MOD_ATTN_KERNEL) on the bench step at the BASELINE shapes, after the variant tests
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attn_pair.py -q -x --timeout 120 > gpurun_out/pytest_var.log 2>&1; echo var_rc=$?; tail -3 gpurun_out/pytest_var.log
for c in ${CONFIGS:-cogvideox-5b hunyuanvideo-720p}; do for kk in ${KERNELS:-single dual single dual}; do
MOD_ATTN_KERNEL=$kk timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bvb.log 2>&1
python - <<PY
import json
for l in open('gpurun_out/bvb.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$c', '$kk', {k:d[k] for k in ('value','attn_ms','attn_tflops')}, d['clocks']['sm_mhz'])
    elif 'rror' in l: print(l[:200])
PY
done; done
