# ncu evidence for profiles/ (round 1): launch list of bench steps + --set full captures of the top kernels.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
KREG='regex:attn_fwd|pool_kernel|score_tc_kernel|softmax_norm|project_kernel|reduce_rhs|solve_|merge_kernel|roll_kernel|select_kernel|count_kernel|write_kernel|keep_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KREG" -c 300 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1; echo launches_rc=$?
for K in attn_fwd pool_kernel score_tc_kernel solve_partial project_kernel select_kernel write_kernel count_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/full_$K -f $B > gpurun_out/ncu_full_$K.log 2>&1; echo ${K}_rc=$?
done
