mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attn_pair.py -q -x --timeout 120 > gpurun_out/pytest_pair.log 2>&1; echo pair_rc=$?; tail -2 gpurun_out/pytest_pair.log
MOD_ATTN_KERNEL=pair MOD_ATTN_DEBUG=16 python scripts/attn_trace.py 2>&1 | grep -v Warn | tail -1; cp gpurun_out/trace.txt gpurun_out/trace_pair.txt
for rep in 1 2; do for kk in single pair; do MOD_ATTN_KERNEL=$kk timeout 100 python scripts/attn_micro.py 2>&1 | grep '^{' | sed "s/^/$kk /"; done; done
