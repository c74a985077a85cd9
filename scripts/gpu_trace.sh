mkdir -p gpurun_out
for d in 19 16; do MOD_ATTN_DEBUG=$d python scripts/attn_trace.py 2>&1 | grep -v Warn | tail -2; cp gpurun_out/trace.txt gpurun_out/trace_$d.txt; done
for d in 0 1 2 3; do MOD_ATTN_DEBUG=$d python scripts/attn_micro.py 2>&1 | grep '^{'; done
