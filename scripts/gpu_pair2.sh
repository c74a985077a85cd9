# CTA-pair K4 (MOD_ATTN_KERNEL=pair2) vs the default kernel: bench step at Hunyuan / Wan, dense mode
mkdir -p gpurun_out
for c in hunyuanvideo-720p wan2.1-14b-720p; do for kk in single pair2 single pair2; do
MOD_ATTN_KERNEL=$kk timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bp2.log 2>&1
python - <<PY
import json
for l in open('gpurun_out/bp2.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$c', '$kk', {k:d[k] for k in ('value','attn_ms','attn_tflops')}, d['clocks']['sm_mhz'])
    elif 'rror' in l: print(l[:200])
PY
done; done
for kk in single pair2; do MOD_ATTN_KERNEL=$kk HEADS=8 timeout 120 python scripts/attn_dense_time.py 2>&1 | grep "^{" | sed "s/^/dense $kk /" | cut -c1-200; done
