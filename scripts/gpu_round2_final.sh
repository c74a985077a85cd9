# round-2 closing measurement set: bench (default flags), ncu launch list + K4 full capture + traffic json,
# K1 score kernels full captures, CogVideoX / Wan lines
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; grep "^{" gpurun_out/bench_full.log | tail -1 | cut -c1-300
KERNS="attn_fwd score_kernel split_kernel pool_kernel solve_stream project_kernel" bash scripts/profile_r2.sh
python scripts/k4_traffic_from_ncu.py gpurun_out/full_attn_fwd.ncu-rep hunyuanvideo-720p 24 "ncu --set full capture of the bench step's K4 launch (scripts/profile_r2.sh)"
cp profiles/k4_traffic.json gpurun_out/k4_traffic.json
rm -f gpurun_out/bench_configs.jsonl
for c in cogvideox-5b wan2.1-14b-720p; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e >> gpurun_out/bench_configs.jsonl 2> gpurun_out/bc_$c.err || tail -3 gpurun_out/bc_$c.err; done
timeout 600 python bench.py > gpurun_out/bench_full2.log 2>&1; grep "^{" gpurun_out/bench_full2.log | tail -1 | cut -c1-300
