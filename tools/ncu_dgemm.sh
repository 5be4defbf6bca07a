#!/bin/bash
# ncu --set full of the config-3 A*G DGEMM (k_dgemm_tm) on tools/gemm_tma_check.py's workload.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/gemm_tma_check.py > gpurun_out/plain_dgemm.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:k_dgemm_tm -s 2 -c 1 -o gpurun_out/ncu_dgemm -f \
    python tools/gemm_tma_check.py > gpurun_out/ncu_dgemm.log 2>&1
tail -1 gpurun_out/ncu_dgemm.log
