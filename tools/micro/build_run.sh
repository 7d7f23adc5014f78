#!/bin/bash
# Build a micro test here and run it on the GPU box: tools/micro/build_run.sh tma_test [filter]
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. -I../../paper_2604_07276_b200/csrc "$1.cu" -o "$1" 2>&1 | grep -E "error" && exit 1
cd ../..
/usr/local/graft/bin/gpurun --timeout 300 -- "cd tools/micro && timeout 120 ./$1"
