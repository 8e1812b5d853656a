#!/bin/bash
# Build and run the arithmetic-pipe microbenchmarks on the GPU box (DESIGN section 5 numbers):
#   bash tools/microbench/run.sh > gpurun_out/microbench.txt
set -e
D=$(dirname "$0")
for f in int_roofline fp_modmul mix_pipes shfl_vs_smem cluster_ntt; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/$f $D/$f.cu
  echo "== $f"
  /tmp/$f
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
