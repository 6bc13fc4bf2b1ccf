set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_baseline.py tests/test_gpu_weights.py tests/test_gpu_parity.py tests/test_sharded.py tests/test_multigpu.py -m gpu -q -p no:cacheprovider > gpurun_out/t14.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/t14.log
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; }
for w in "c2 --batch 1" "c3 --batch 1" "c4 --batch 1"; do set -- $w; timeout 900 python bench.py --workload $w --no-cpu-baseline > "gpurun_out/b14_$1.log" 2>&1; show "gpurun_out/b14_$1.log" "$1B1"; done
HYRE_SMALL=0 timeout 600 python bench.py --workload c3 --batch 1 --no-cpu-baseline > gpurun_out/b14_c3_nosmall.log 2>&1; show gpurun_out/b14_c3_nosmall.log c3B1_nosmall
