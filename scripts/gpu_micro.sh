mkdir -p gpurun_out
for d in 0 1 2 3; do MOD_ATTN_DEBUG=$d timeout 300 python scripts/attn_micro.py $1; done 2>&1 | tee gpurun_out/micro.log
