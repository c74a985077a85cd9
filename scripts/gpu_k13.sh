# K1-K3 iteration: parity of stats / fit / update / plan, the bench step's overhead, a launch list
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py tests/test_gpu_c_example.py -x -q --timeout 200 -k "${K:-stats or fit or update or plan or solver or keep or predict or schedule or example}" > gpurun_out/pytest_k13.log 2>&1; tail -15 gpurun_out/pytest_k13.log | grep -v "^$"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense > gpurun_out/bench_k13.log 2>&1
grep "^{" gpurun_out/bench_k13.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('attn_ms', d['attn_ms'], 'overhead', d['pipeline_overhead_ms'])" || tail -3 gpurun_out/bench_k13.log
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
KREG='regex:pool_kernel|score_|softmax_norm|project_|reduce_rhs|solve_|merge_kernel|roll_kernel|select_kernel|count_kernel|write_kernel|keep_kernel'
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KREG" -c 60 --csv --log-file gpurun_out/launches_k13.csv $B > /dev/null 2>&1; echo ncu_rc=$?
