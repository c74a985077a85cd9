mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 1 -c 1 -o gpurun_out/k4_wide -f python scripts/k4_run.py ${CFG:-hunyuanvideo-720p} wide 2 > gpurun_out/ncu_k4_wide.log 2>&1; echo rc=$?
