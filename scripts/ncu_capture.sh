#!/bin/bash
# One `ncu --set full` capture of the dominant kernel per config (run alone on one GPU).
# Output: gpurun_out/<tag>.ncu-rep ; summarise with scripts/ncu_summary.py
set -u
cap() {  # tag workload format kernel-regex
  ncu --set full --import-source on --clock-control none -k "regex:$4" -s 3 -c 1 -o "gpurun_out/$1" \
    python scripts/profile_kernel.py --workload "$2" --format "$3" --reps 2 > "gpurun_out/$1.log" 2>&1
}
cap r01_ncu_c5_csr5 C5 csr5 k_csr5_warp_s
cap r01_ncu_c4_csr5 C4 csr5 k_csr5_warp_s
cap r01_ncu_c4_csr C4 csr k_spmv_chunk
cap r01_ncu_c3_ell C3 ell k_spmv_ell
cap r01_ncu_c2_ell C2 ell k_spmv_ell
