#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the GPU
# parity tests that exercise shared-memory transposes, the radix sort's
# decoupled look-back, cross-block carry fix-ups and the fused peer push.
#   bash scripts/sanitize.sh [outdir]      (on the GPU box; logs per tool)
# PYTORCH_NO_CUDA_MEMORY_CACHING=1 gives every torch tensor its own
# allocation, so out-of-bounds accesses past a tensor are caught too.
set -u
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
TESTS=(
  "tests/test_gpu_parity.py::test_every_case_matches_reference"
  "tests/test_gpu_parity.py::test_canonicalize_many_tiles"
  "tests/test_gpu_parity.py::test_wide_rows_sell_hyb"
  "tests/test_gpu_parity.py::test_random_sweep_against_oracle"
  "tests/test_gpu_p2p.py::test_push_rows_to_local_peers"
  "tests/test_gpu_p2p.py::test_fused_spmv_push_to_local_peers"
  "tests/test_gpu_p2p.py::test_power_iteration_graph_replay_identical"
  "tests/test_gpu_dispatch.py::test_norm_scale_kernel"
  "tests/test_gpu_dispatch.py::test_bind_bit_identical"
  "tests/test_gpu_relabel.py"
)
for tool in memcheck racecheck synccheck initcheck; do
  extra=()
  [ "$tool" = memcheck ] && extra=(--leak-check no)
  [ "$tool" = racecheck ] && extra=(--racecheck-report hazard)
  timeout 3000 compute-sanitizer --tool "$tool" "${extra[@]}" --target-processes all \
    --print-limit 200 --error-exitcode 17 \
    python -m pytest -q -x -m gpu -p no:cacheprovider "${TESTS[@]}" > "$out/$tool.log" 2>&1
  echo "$tool exit $?" | tee -a "$out/summary.txt"
  grep -E "ERROR SUMMARY|passed|failed" "$out/$tool.log" | tail -3 | tee -a "$out/summary.txt"
done
