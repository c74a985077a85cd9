#!/bin/bash
# GPU check: build, the -m gpu suite, one bench line per K4 schedule
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build --force > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for kk in ${KERNELS:-default splitkv}; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --attn-kernel $kk > gpurun_out/bench_$kk.log 2>&1
  grep "^{" gpurun_out/bench_$kk.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$kk', 'value', d['value'], 'attn_ms', d['attn_ms'], 'frac', d['roofline']['frac'], 'kernel', d['roofline']['kernel'], 'dense', d['dense_ms'], 'e2e', d['e2e'] and d['e2e']['ms_per_step'], 'clk', d['clocks'])" || tail -5 gpurun_out/bench_$kk.log
done
