# round-end measurement set: all GPU tests, the default bench line (Hunyuan), the other BASELINE
# configs (Wan, CogVideoX), the reference arm (oracle on host cores)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/pytest_gpu.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_full.log | cut -c1-400
for c in wan2.1-14b-720p cogvideox-5b; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.log 2>&1; echo ${c}_rc=$?; tail -1 gpurun_out/bench_$c.log | cut -c1-300
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-300
