mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "not attention" > gpurun_out/pytest_nonattn.log 2>&1; echo rc=$?
tail -30 gpurun_out/pytest_nonattn.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -20 gpurun_out/bench.log
