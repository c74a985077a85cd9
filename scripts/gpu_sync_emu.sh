python -m paper_2601_11641_b200.build > /dev/null 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$? $(tail -1 gpurun_out/sanitize_synccheck.log)"
timeout 300 python -m pytest tests/test_gpu_attn_pair.py -q -x --timeout 200 2>&1 | tail -1
NOBENCH=1 VARIANTS="k4t_base k4t_e2_1 k4t_e3_1 k4t_e3_2" bash scripts/gpu_k4_ab_r2.sh
