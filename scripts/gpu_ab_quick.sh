# quick K4 check: attention parity + short and sustained micro A/B of the kernel variants
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "attention or attn or pair" > gpurun_out/pytest_attn.log 2>&1; echo attn_rc=$?; tail -2 gpurun_out/pytest_attn.log
for rep in 1 2; do for kk in ${KERNELS:-single pair}; do MOD_ATTN_KERNEL=$kk timeout 100 python scripts/attn_micro.py 2>&1 | grep '^{' | sed "s/^/$kk /"; done; done
for kk in ${KERNELS:-single pair}; do MOD_ATTN_KERNEL=$kk REPS=300 timeout 200 python scripts/attn_micro.py 2>&1 | grep '^{' | sed "s/^/sustained $kk /"; done
