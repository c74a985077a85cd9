# --set full capture of one kernel (KNAME) from a short bench run
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KNAME -s 3 -c 1 -o gpurun_out/one_$KNAME -f $B > /dev/null 2>&1; echo rc=$?
