# bench.py step with K1 beside K4 (default) vs --serial-k1, alternating R rounds (attention-only lines)
for r in $(seq 1 ${R:-3}); do
  for m in overlap serial; do
    extra=""; [ $m = serial ] && extra="--serial-k1"
    timeout 300 python bench.py --config ${CFG:-hunyuanvideo-720p} --steps ${STEPS:-30} --warmup 5 --no-cpu --no-e2e --no-dense $extra > gpurun_out/bk1_$m.log 2>&1
    grep "^{" gpurun_out/bk1_$m.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$r $m', d['value'], d['ms_per_step'], d['attn_ms'], d['pipeline_overhead_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bk1_$m.log
  done
done
