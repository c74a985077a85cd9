#!/bin/bash
# K4 iteration: variant tests, trace of the default kernel, bench A/B (default vs splitkv)
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_attn_pair.py -x -q > gpurun_out/pytest_pair.log 2>&1; tail -3 gpurun_out/pytest_pair.log
MODDIT_LIB_OVERRIDE=_variants/k4trace/libmoddit.so timeout 300 python scripts/k4_trace.py ${CFG:-hunyuanvideo-720p} default > gpurun_out/k4_trace.json 2> gpurun_out/k4_trace.err
python -c "
import json; d=json.load(open('gpurun_out/k4_trace.json')); t=d.pop('traced'); print(d)
for r in t[:3]: print(r)"
tail -2 gpurun_out/k4_trace.err
for kk in ${KERNELS:-default splitkv default}; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --attn-kernel $kk > gpurun_out/bench_$kk.log 2>&1
  python - "$kk" <<'PY'
import json,sys
kk=sys.argv[1]
for l in open(f"gpurun_out/bench_{kk}.log"):
    if l.startswith("{"):
        d=json.loads(l); print(kk, "attn_ms", d["attn_ms"], "attn_tflops", d["attn_tflops"], "frac", d["roofline"]["frac"], "dense", d["dense_ms"].get("ours_all_ones_csr"), "cudnn", d["dense_ms"].get("cudnn"), "clk", d["clocks"])
PY
done
