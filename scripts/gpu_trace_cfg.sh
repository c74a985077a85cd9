mkdir -p gpurun_out
MOD_ATTN_DEBUG=16 python scripts/attn_trace.py ${CFG:-cogvideox-5b} 2>&1 | grep -v Warn | tail -1; cp gpurun_out/trace.txt gpurun_out/trace_${CFG:-cogvideox-5b}.txt
