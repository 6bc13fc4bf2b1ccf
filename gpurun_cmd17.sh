set -u
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest17.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest17.log
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['value']), d.get('reruns'))"; }
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b17_c3.log 2>&1; show gpurun_out/b17_c3.log c3
for w in "c2 --batch 1" "c3 --batch 1" "c4 --batch 1"; do set -- $w; timeout 900 python bench.py --workload $w --no-cpu-baseline > "gpurun_out/b17_$1.log" 2>&1; show "gpurun_out/b17_$1.log" "$1B1"; done
