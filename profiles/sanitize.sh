#!/bin/bash
# compute-sanitizer passes over small GPU parity cases (one python process
# per tool); summaries -> gpurun_out/sanitize_<tool>.log
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
SEL='test_tensor_core_batch_matches_oracle or test_fused_cnf_eligibility_bitexact or test_bucket_selection or test_batch_execution_matches_single or test_candidate_overflow_recovers or test_match_all_tensor_core_batch or test_quantized_preselection or test_term_only or test_prefilter_keeps_exact_order'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 0 \
    --target-processes all python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/sanitize_$tool.log) summaries"
  grep -E "ERROR SUMMARY|passed|failed|RACECHECK SUMMARY" gpurun_out/sanitize_$tool.log | sort | uniq -c | head -8
done
