mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
for K in ${KERNS:-project_kernel solve_stream}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/full_$K -f $B > gpurun_out/ncu_full_$K.log 2>&1; echo ${K}_rc=$?
done
