mkdir -p gpurun_out
for d in ${DBGS:-0 1 4 8 12}; do MOD_ATTN_DEBUG=$d timeout 100 python scripts/attn_micro.py $1; done 2>&1 | tee gpurun_out/micro.log
