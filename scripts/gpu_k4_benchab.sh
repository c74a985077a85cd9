# bench attention-time A/B of library variants (_variants/NAME), alternating, R rounds
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for r in $(seq 1 ${R:-2}); do
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset MODDIT_LIB_OVERRIDE; else export MODDIT_LIB_OVERRIDE=_variants/$v/libmoddit.so; fi
  timeout 300 python bench.py --config ${CFG:-hunyuanvideo-720p} --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense --attn-kernel ${KK:-default} > gpurun_out/bab_$v.log 2>&1
  grep "^{" gpurun_out/bab_$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$r $v', 'attn_ms', d['attn_ms'], 'tflops', d['attn_tflops'], 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bab_$v.log
done; done
