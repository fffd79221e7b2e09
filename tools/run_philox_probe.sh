#!/bin/bash
# Build and run the Philox4x64-10 throughput probe (bit-exact uniforms/s ceiling of K1).
set -e
cd "$(dirname "$0")/probes"
/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o philox_probe philox_probe.cu
./philox_probe
