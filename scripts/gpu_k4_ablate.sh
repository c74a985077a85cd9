#!/bin/bash
# A/B of K4 trace builds (_variants/k4t_*): cycles per block, effective clock, pipeline intervals
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_attn_pair.py -x -q > gpurun_out/pytest_pair.log 2>&1; tail -2 gpurun_out/pytest_pair.log
for n in ${VARIANTS:-$(ls _variants | grep k4t_)}; do
  MODDIT_LIB_OVERRIDE=_variants/$n/libmoddit.so timeout 300 python scripts/k4_trace.py ${CFG:-hunyuanvideo-720p} default > gpurun_out/abl_$n.json 2> gpurun_out/abl_$n.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/abl_$n.json')); t=d.pop('traced'); print('$n', {k:d[k] for k in ('ms','eff_clock_ghz','cycles_fixed_per_cta','cycles_per_block')})
r=t[0]; print('   ', {k:v for k,v in r.items() if k not in ('cta',)})" || tail -3 gpurun_out/abl_$n.err
done
