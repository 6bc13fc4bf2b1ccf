set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baseline.py tests/test_gpu_parity.py tests/test_gpu_weights.py -m gpu -q -x -p no:cacheprovider -k "c3_shape or tensor_core or fused or match_all or candidate_overflow or indistinguishable or row_variants or weighted_cnf or quant_preselection_batches or k_above" > gpurun_out/t8.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t8.log
bash profiles/k3_sweep.sh "bias" "nobias HYRE_TC_BIAS=0" 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b8.log 2>&1; grep '^{' gpurun_out/b8.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['value']), 'inflight2', round(d['inflight2']['value']), d['parity'] if 'parity' in d else '')"
ncu --set full --clock-control none -k regex:"select_kernel|small_topk" -c 4 -o gpurun_out/r02_c1_small python bench.py --workload c1 --batch 1 --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "ncu c1 rc=$?"
