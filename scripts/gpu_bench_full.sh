mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_full.log | cut -c1-3000
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-1500
