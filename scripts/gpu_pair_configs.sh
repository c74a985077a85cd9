# single vs pair K4 at the three BASELINE shapes (bench step, attention timed alone)
mkdir -p gpurun_out
for c in cogvideox-5b wan2.1-14b-720p hunyuanvideo-720p; do for kk in single pair single pair; do
MOD_ATTN_KERNEL=$kk timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bpc.log 2>&1
python - <<PY
import json
for l in open('gpurun_out/bpc.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$c', '$kk', {k:d[k] for k in ('value','attn_ms','attn_tflops')}, d['clocks']['sm_mhz'])
PY
done; done
