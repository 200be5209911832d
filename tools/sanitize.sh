#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the small GPU unit
# tests: every library kernel family (operators, fused elimination pass, pivot
# commit, fsub, normalise, sketches, projected-solve cooperative kernel,
# sharded loops with the in-process communicator).  Summaries -> gpurun_out/sanitize_*.txt
cd "$(dirname "$0")/.."
T="tests/test_gpu_parity.py::test_slslu_tomography_vs_reference_bitwise tests/test_gpu_parity.py::test_scmrh_dense_vs_reference tests/test_gpu_parity.py::test_sketches tests/test_gpu_parity.py::test_fp32_deblur_vs_oracle32 tests/test_gpu_parity.py::test_edge_cases_vs_reference tests/test_gpu_parity.py::test_rank_fallback_min_norm_vs_reference tests/test_gpu_parity.py::test_sampled_pivoting_and_unsketched_vs_reference tests/test_gpu_stepper.py tests/test_gpu_local_ranks.py::test_local_ranks_slslu_bitwise"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest $T -q -x -p no:cacheprovider -k "not 8 and not 4" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
  tail -4 gpurun_out/sanitize_$tool.txt
done
