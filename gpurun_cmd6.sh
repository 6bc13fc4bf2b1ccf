set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_weights.py tests/test_gpu_baseline.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "weight or c1_full or equals_single or hybrid_execution or acceptance or k_larger or zero_query or batch_execution" > gpurun_out/t6.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/t6.log
for w in "c1 --batch 1" "c2 --batch 1"; do set -- $w; timeout 600 python bench.py --workload $w --no-cpu-baseline > "gpurun_out/b6_$1.log" 2>&1; grep '^{' "gpurun_out/b6_$1.log" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['p50_ms'], d.get('stages_ms'), d.get('e2e',{}).get('value'))"; done
HYRE_SMALL=0 timeout 600 python bench.py --workload c1 --batch 1 --no-cpu-baseline > gpurun_out/b6_c1_nosmall.log 2>&1; grep '^{' gpurun_out/b6_c1_nosmall.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 nosmall', d['value'], d['p50_ms'], d.get('stages_ms'))"
