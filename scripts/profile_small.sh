mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:${KREG:-pool_kernel|score_kernel|project_kernel|reduce_rhs|solve_partial|solve_reduce|merge_kernel|roll_kernel|select_kernel|count_kernel|write_kernel}" -c 200 --csv --log-file gpurun_out/launches_small.csv $B > /dev/null 2>&1; echo rc=$?
