#!/bin/bash
# Build + run the batched-kernel phase timer (needs the library built first).
cd "$(dirname "$0")"
R=../../paper_1212_4560_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -I$R/csrc --expt-relaxed-constexpr \
    -o b64_prof b64_prof.cu -L$R/lib -lrl_b200 -Xlinker -rpath -Xlinker '$ORIGIN/'$R/lib && ./b64_prof
