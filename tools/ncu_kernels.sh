#!/bin/bash
# One ncu --set full capture per kernel of interest, each on the smallest
# workload of tools/prof_kernels.py that launches it; the plain run of that workload exits 0 first.
# Reports land in gpurun_out/ncu_<name>.ncu-rep; tools/ncu_summarize.py turns them into
# profiles/r02_ncu_kernels.json.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cap() { # name workload regex skip
  python tools/prof_kernels.py "$2" > gpurun_out/plain_$1.log 2>&1 &&
  ncu --set full --import-source on --clock-control none -k "regex:$3" -s "$4" -c 1 \
      -o "gpurun_out/ncu_$1" -f python tools/prof_kernels.py "$2" > "gpurun_out/ncu_$1.log" 2>&1
  echo "$1: $(tail -1 gpurun_out/ncu_$1.log)"
}
cap batched     c2      "k_batched_circ64"  1
cap hh2         hh      "k_hh2_onepass"     1
cap sparse      sparse  "k_sparse_right4"   1
cap sparseplan  sparse  "k_sparse_plan"     1
cap circfft     circfft "k_circ_fft8k"      1
cap cholinv     c4      "k_chol_inv"        6
cap bidiag      c4      "k_bidiag_sv"       2
cap rf_dgemm    c4      "k_dgemm_tm<128, 72"   1
cap rf_dgemm_qta c4     "k_dgemm_tm<72, 128"   1
cap gen_chunks  rng     "k_gen_chunks"      1
cap diag_lu     lu      "k_diag_lu"         64
cap panel_trsm  lu      "k_panel_trsm"      64
cap trsv_wave   lu      "k_trsv_wave"       2
cap lu_dgemm    lu      "k_dgemm_tm<128, 64"   2
