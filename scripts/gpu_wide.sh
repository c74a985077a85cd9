mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -u -m pytest tests/test_gpu_attn_pair.py -x -q --timeout 120 -k "wide" > gpurun_out/pytest_wide.log 2>&1; tail -3 gpurun_out/pytest_wide.log
for cfg in hunyuanvideo-720p cogvideox-5b; do
for kk in default wide; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-e2e --attn-kernel $kk > gpurun_out/bw_${cfg}_$kk.log 2>&1
  grep "^{" gpurun_out/bw_${cfg}_$kk.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$cfg $kk attn_ms', d['attn_ms'], 'tflops', d['attn_tflops'], 'frac', d['roofline']['frac'], 'dense', d['dense_ms'].get('ours_all_ones_csr'), d['dense_ms'].get('cudnn'), 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bw_${cfg}_$kk.log
done; done
