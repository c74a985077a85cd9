mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu > gpurun_out/bench_quick.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/bench_quick.log | cut -c1-1500
