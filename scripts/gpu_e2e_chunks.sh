mkdir -p gpurun_out
for c in 8 12 24; do timeout 400 python bench.py --steps 5 --warmup 3 --no-dense --no-cpu --e2e-chunks $c > gpurun_out/bench_e2e_$c.log 2>&1
python - <<PY
import json
for l in open('gpurun_out/bench_e2e_$c.log'):
    if l.startswith('{'):
        d=json.loads(l); print($c, d['e2e']['ms_per_step'], d['e2e']['value'], d['attn_tflops'])
PY
done
