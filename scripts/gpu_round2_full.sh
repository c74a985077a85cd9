# round-2 measurement set: gpu tests, bench (default flags), ncu launch list + K4 full capture, traffic json
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -u -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; grep "^{" gpurun_out/bench_full.log | tail -1 | cut -c1-600
bash scripts/profile_r2.sh
python scripts/k4_traffic_from_ncu.py gpurun_out/full_attn_fwd.ncu-rep hunyuanvideo-720p 24 "ncu --set full capture of the bench step's K4 launch (scripts/profile_r2.sh)"
cp profiles/k4_traffic.json gpurun_out/k4_traffic.json
