# A/B of a K4 bring-up switch (MOD_ATTN_DEBUG=$DBG vs 0) on the bench step at the BASELINE shapes
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "attention or attn or pair" > gpurun_out/pytest_attn.log 2>&1; echo attn_rc=$?; tail -1 gpurun_out/pytest_attn.log
for c in ${CONFIGS:-cogvideox-5b hunyuanvideo-720p}; do for d in 0 $DBG 0 $DBG; do
MOD_ATTN_DEBUG=$d timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bab.log 2>&1
python - <<PY
import json
for l in open('gpurun_out/bab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$c', 'dbg=$d', {k:d[k] for k in ('value','attn_ms','attn_tflops')}, d['clocks']['sm_mhz'])
PY
done; done
