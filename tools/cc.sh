#!/bin/bash
# compile-check one CUDA source with ptxas info (dev helper): tools/cc.sh genp.cu
cd "$(dirname "$0")/../paper_1212_4560_b200/csrc" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -I../../include -I. -Xptxas -v -c "$1" -o "/tmp/$(basename "$1" .cu).o" 2>&1 | grep -E "error|warning|registers|spill"
