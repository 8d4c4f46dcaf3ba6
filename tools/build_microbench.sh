#!/bin/bash
# Build the microbenchmarks into tools/bin (git-ignored; they travel to the GPU box with gpurun).
set -e
cd "$(dirname "$0")"
mkdir -p bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o bin/f64_latency f64_latency.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/globaltimer_resolution globaltimer_resolution.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/warp_min_rounds warp_min_rounds.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/zero_copy zero_copy.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/sysmem_writes sysmem_writes.cu
