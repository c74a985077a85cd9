# K4 variant A/B: parity (attention tests) per non-trace variant, trace per trace variant, bench per variant
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for v in ${TESTVARIANTS}; do
  MODDIT_LIB_OVERRIDE=_variants/$v/libmoddit.so timeout 300 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_attn_pair.py -x -q -k "attention or attn" --timeout 120 > gpurun_out/pytest_attn_$v.log 2>&1; echo "$v $(tail -1 gpurun_out/pytest_attn_$v.log)"
done
NOBENCH=1 bash scripts/gpu_k4_ab_r2.sh
for v in ${TESTVARIANTS} default; do
  if [ $v = default ]; then unset MODDIT_LIB_OVERRIDE; else export MODDIT_LIB_OVERRIDE=_variants/$v/libmoddit.so; fi
  timeout 240 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$v.log 2>&1
  grep "^{" gpurun_out/bench_$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$v attn_ms', d['attn_ms'], 'tflops', d['attn_tflops'], 'frac', d['roofline']['frac'], 'dense', d['dense_ms'], 'clk', d['clocks'])" || tail -3 gpurun_out/bench_$v.log
done
