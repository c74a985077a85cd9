#!/bin/bash
# K4 schedule A/B: build, variant parity tests, then the bench step with each schedule
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build --force > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_attn_pair.py tests/test_gpu_parity.py -x -q ${PYTEST_ARGS} > gpurun_out/pytest_k4.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_k4.log
tail -5 gpurun_out/pytest_k4.log
for kk in ${KERNELS:-default splitkv default splitkv}; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --attn-kernel $kk > gpurun_out/bench_$kk.log 2>&1
  python - "$kk" <<'PY'
import json,sys
kk=sys.argv[1]
for l in open(f"gpurun_out/bench_{kk}.log"):
    if l.startswith("{"):
        d=json.loads(l); print(kk, "attn_ms", d["attn_ms"], "attn_tflops", d["attn_tflops"], "frac", d["roofline"]["frac"], "dense", d["dense_ms"].get("ours_all_ones_csr"), "cudnn", d["dense_ms"].get("cudnn"), "clk", d["clocks"])
PY
done
