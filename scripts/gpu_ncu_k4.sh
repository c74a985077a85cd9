#!/bin/bash
# one ncu --set full capture of the K4 kernel on the bench workload (plus a pipe-utilisation csv)
mkdir -p gpurun_out
python -m paper_2601_11641_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
KK=${KK:-default}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 1 -c 1 -o gpurun_out/k4_$KK -f python scripts/k4_run.py ${CFG:-hunyuanvideo-720p} $KK 2 > gpurun_out/ncu_k4_$KK.log 2>&1
tail -3 gpurun_out/ncu_k4_$KK.log
ncu -i gpurun_out/k4_$KK.ncu-rep --page raw --csv > gpurun_out/k4_${KK}_raw.csv 2>/dev/null
ncu -i gpurun_out/k4_$KK.ncu-rep --page source --csv > gpurun_out/k4_${KK}_source.csv 2>/dev/null
ls -la gpurun_out/k4_$KK*
