#!/bin/bash
# K4 A/B (round 2): trace variants (_variants/k4t_*) -> cycles per block, clock, pipeline intervals;
# then the shipped build's bench line (attention only)
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for n in ${VARIANTS:-$(ls _variants | grep k4t_)}; do
  MODDIT_LIB_OVERRIDE=_variants/$n/libmoddit.so TIMELINE=1 timeout 120 python scripts/k4_trace.py ${CFG:-hunyuanvideo-720p} default > gpurun_out/abl_$n.txt 2> gpurun_out/abl_$n.err
  head -1 gpurun_out/abl_$n.txt | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); t=d.pop('traced'); print('$n', {k:d[k] for k in ('ms','eff_clock_ghz','cycles_fixed_per_cta','cycles_per_block')})
r=t[0] if t else {}; print('   ', {k:v for k,v in r.items() if k not in ('cta',)})" || tail -3 gpurun_out/abl_$n.err
done
if [ -z "$NOBENCH" ]; then
timeout 240 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_ab.log 2>&1
grep "^{" gpurun_out/bench_ab.log | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('bench attn_ms', d['attn_ms'], 'tflops', d['attn_tflops'], 'frac', d['roofline']['frac'], 'dense', d['dense_ms'], 'clk', d['clocks'])" || tail -5 gpurun_out/bench_ab.log
fi
