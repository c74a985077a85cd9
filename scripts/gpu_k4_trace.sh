#!/bin/bash
# K4 trace build: per-CTA spans + per-block pipeline intervals (scripts/k4_trace.py)
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
[ -f _variants/k4trace/libmoddit.so ] || EXTRA_NVCC=-DMOD_K4_TRACE bash scripts/build_variant.sh k4trace
for kk in ${KERNELS:-default}; do
MODDIT_LIB_OVERRIDE=_variants/k4trace/libmoddit.so timeout 300 python scripts/k4_trace.py ${CFG:-hunyuanvideo-720p} $kk > gpurun_out/k4_trace_$kk.json 2> gpurun_out/k4_trace_$kk.err
cat gpurun_out/k4_trace_$kk.json; tail -3 gpurun_out/k4_trace_$kk.err
done
timeout 600 python -m pytest tests/test_gpu_attn_pair.py -x -q > gpurun_out/pytest_pair.log 2>&1; tail -3 gpurun_out/pytest_pair.log
