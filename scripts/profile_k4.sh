mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-dense --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/k4_full -f $B > gpurun_out/ncu_k4_stdout.log 2>&1; echo k4_rc=$?
