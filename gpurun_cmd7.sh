set -u
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest7.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/gputest7.log
for v in "pdl" "nopdl HYRE_PDL=0"; do set -- $v; env ${2:-X=1} timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b7_$1.log 2>&1; grep '^{' gpurun_out/b7_$1.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['value']), 'inflight2', round(d['inflight2']['value']))"; done
for w in "c1 --batch 1" "c2 --batch 1" "c2 --batch 256"; do set -- $w; timeout 600 python bench.py --workload $w --no-cpu-baseline > "gpurun_out/b7_$1_$3.log" 2>&1; grep '^{' "gpurun_out/b7_$1_$3.log" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 B=$3', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; done
