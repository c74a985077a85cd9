#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mma_probe scripts/micro/mma_probe.cu && timeout 120 /tmp/mma_probe | tee gpurun_out/mma_probe.log
