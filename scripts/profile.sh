# ncu evidence for profiles/: launch list of one bench step and --set full captures of K4 and K1.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
KREG='regex:attn_fwd|pool_kernel|score_kernel|project_kernel|reduce_rhs|solve_kernel|merge_kernel|roll_kernel|predict_kernel|keep_kernel|dense_mask'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KREG" -c 200 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/k4_full -f $B > gpurun_out/ncu_k4_stdout.log 2>&1; echo k4_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pool_kernel -s 3 -c 1 -o gpurun_out/k1_pool_full -f $B > gpurun_out/ncu_k1_stdout.log 2>&1; echo k1_rc=$?
ls -la gpurun_out
