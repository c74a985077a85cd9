# ncu evidence for profiles/r2: launch list of two bench steps (per-launch time + DRAM bytes) and
# --set full captures of the kernels named in $KERNS (default: K4 only).
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
KREG='regex:attn_|pool_kernel|score_|softmax_norm|project_|reduce_rhs|solve_|merge_kernel|roll_kernel|select_kernel|count_kernel|write_kernel|keep_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KREG" -c 300 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1; echo launches_rc=$?
for K in ${KERNS:-attn_fwd}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/full_$K -f $B > gpurun_out/ncu_full_$K.log 2>&1; echo ${K}_rc=$?
done
