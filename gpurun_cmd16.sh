set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baseline.py tests/test_gpu_parity.py tests/test_gpu_weights.py -m gpu -q -x -p no:cacheprovider -k "c3_shape or tensor_core or fused or candidate_overflow or indistinguishable or row_variants or weighted_cnf or quant_preselection_batches or k_above or segmented" > gpurun_out/t16.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t16.log
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()}, d.get('reruns'), 'e2e', round(d['e2e']['value']), 'inflight2', round(d.get('inflight2',{}).get('value',0)))"; }
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b16_c3.log 2>&1; show gpurun_out/b16_c3.log c3
HYRE_TC_SAMPLE_CC=0 timeout 600 python bench.py --no-cpu-baseline --inflight 1 > gpurun_out/b16_c3_tcs.log 2>&1; show gpurun_out/b16_c3_tcs.log c3_tcsample
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02e_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "launches rc=$?"
