bash profiles/k3_sweep.sh "merged" "merged_noCNF HYRE_TC_DEBUG=4" "merged_mmaonly HYRE_TC_DEBUG=6" 2>&1
timeout 900 python -m pytest tests/test_gpu_baseline.py tests/test_gpu_parity.py -m gpu -q -x -k "c3_shape or tensor_core or fused or variants or quant or prefilter" > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
