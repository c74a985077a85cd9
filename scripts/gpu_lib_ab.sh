# A/B of the working-tree library against _variants/$BASE on the bench step (attention timed alone)
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 -k "attention or attn or pair or schedule or exact or quant" > gpurun_out/pytest_attn.log 2>&1; echo attn_rc=$?; tail -1 gpurun_out/pytest_attn.log
for c in ${CONFIGS:-hunyuanvideo-720p wan2.1-14b-720p}; do for lib in new base new base; do
if [ $lib = base ]; then export MODDIT_LIB_OVERRIDE=_variants/${BASE:-base}/libmoddit.so; else unset MODDIT_LIB_OVERRIDE; fi
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu $EXTRA > gpurun_out/blab.log 2>&1
python - <<PY
import json
for l in open('gpurun_out/blab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$c', '$lib', {k:d[k] for k in ('value','attn_ms','attn_tflops')}, d['clocks']['sm_mhz'])
    elif 'rror' in l: print(l[:200])
PY
done; done
