set -u
mkdir -p gpurun_out
bash profiles/k3_sweep.sh "grouped" "segmented HYRE_CNF_GROUPED=0" "grouped_nocnf HYRE_TC_DEBUG=4" 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest4.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest4.log
timeout 600 python bench.py > gpurun_out/bench4.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench4.log | tail -1 | cut -c1-700
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 --kernel-name-exclude kns=tc_score --error-exitcode 0 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "test_bucket_selection or test_batch_execution_matches_single or test_candidate_overflow_recovers or test_quantized_preselection or test_term_only or test_batched_tbr or batch_scan" > gpurun_out/sanitize_racecheck_nontc.log 2>&1; echo "racecheck rc=$?"; grep -E "SUMMARY|passed|failed" gpurun_out/sanitize_racecheck_nontc.log | tail -3
