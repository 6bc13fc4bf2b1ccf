set -u
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest18.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest18.log
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['value']))"; }
for w in "c3 --batch 1" "c3 --batch 8" "c5 --batch 1 --k 1000"; do set -- $w; timeout 900 python bench.py --workload $w --no-cpu-baseline > "gpurun_out/b18_$1_$3.log" 2>&1; show "gpurun_out/b18_$1_$3.log" "$1B$3"; done
