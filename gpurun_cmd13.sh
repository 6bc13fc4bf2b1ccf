set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baseline.py tests/test_gpu_parity.py tests/test_gpu_weights.py tests/test_sharded.py -m gpu -q -x -p no:cacheprovider -k "c3_shape or tensor_core or fused or match_all or candidate_overflow or indistinguishable or row_variants or weighted or quant_preselection_batches or k_above or c2 or c4 or tied or sharded" > gpurun_out/t13.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t13.log
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()}, 'rr', d.get('reruns'))"; }
timeout 600 python bench.py --no-cpu-baseline --inflight 1 > gpurun_out/b13_c3.log 2>&1; show gpurun_out/b13_c3.log c3
timeout 600 python bench.py --workload c2 --batch 256 --no-cpu-baseline --inflight 1 > gpurun_out/b13_c2.log 2>&1; show gpurun_out/b13_c2.log c2B256
timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b13_c4.log 2>&1; show gpurun_out/b13_c4.log c4B1024
