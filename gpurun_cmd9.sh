set -u
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest9.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/gputest9.log
for w in "c1 --batch 1" "c2 --batch 1" "c3 --batch 1"; do set -- $w; timeout 600 python bench.py --workload $w --no-cpu-baseline > "gpurun_out/b9_$1_$3.log" 2>&1; grep '^{' "gpurun_out/b9_$1_$3.log" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 B=$3', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; done
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 3 -c 1 -o gpurun_out/r02c_tc_main python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "ncu rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "launches rc=$?"
