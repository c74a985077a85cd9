mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 400 python -u -m pytest tests/test_gpu_parity.py -x -v -k "attention" --timeout 120 > gpurun_out/pytest_attn.log 2>&1; grep -E "PASS|FAIL|Timeout|passed|failed" gpurun_out/pytest_attn.log | tail -14
for v in ${TESTVARIANTS}; do
MODDIT_LIB_OVERRIDE=_variants/$v/libmoddit.so timeout 400 python -u -m pytest tests/test_gpu_parity.py -x -q -k "attention" --timeout 120 > gpurun_out/pytest_attn_$v.log 2>&1; echo $v; tail -2 gpurun_out/pytest_attn_$v.log
done
bash scripts/gpu_k4_ab_r2.sh
