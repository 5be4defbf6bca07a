#!/bin/bash
# GPU Box-Muller vs the GPU host's libm on 2^30 random pairs, plus the
# config-3 G (8192^2, stream (20260825, 11)) against the oracle byte for byte.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
  echo "host: $(grep -m1 'model name' /proc/cpuinfo)"
  echo "flags: $(grep -m1 -o -w -E 'fma|avx2' /proc/cpuinfo | sort -u | tr '\n' ' ')"
  echo "libm: $(readlink -f /lib/x86_64-linux-gnu/libm.so.6) $(sha256sum /lib/x86_64-linux-gnu/libm.so.6 | cut -c1-16)"
  t0=$(date +%s.%N)
  paper_1212_4560_b200/lib/bm_libm_check 30
  echo "bm_libm_check 2^30: $(python3 -c "import time; print(round(time.time() - $t0, 1))") s"
  python tools/g_hash.py
} 2>&1 | tee gpurun_out/bm_full.txt
