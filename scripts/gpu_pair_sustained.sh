# sustained (power-capped) A/B of the K4 variants: ~4 s of back-to-back launches each
mkdir -p gpurun_out
for rep in 1 2; do for kk in single pair; do MOD_ATTN_KERNEL=$kk REPS=300 timeout 200 python scripts/attn_micro.py 2>&1 | grep '^{' | sed "s/^/$kk /"; done; done
