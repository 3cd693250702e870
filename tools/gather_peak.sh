#!/bin/bash
# Build and run the random-gather microbenchmark (tools/gather_peak.cu) on the GPU box.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/gather_peak tools/gather_peak.cu
gpurun_out/gather_peak
