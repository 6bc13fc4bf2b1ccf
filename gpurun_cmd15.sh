set -u
mkdir -p gpurun_out
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; }
timeout 600 python bench.py --workload c2 --batch 1 --no-cpu-baseline > gpurun_out/b15_c2b1.log 2>&1; show gpurun_out/b15_c2b1.log c2B1
for v in "d18 HYRE_TC_DEBUG=18" "d10 HYRE_TC_DEBUG=10" "d26 HYRE_TC_DEBUG=26"; do set -- $v; env $2 timeout 900 python bench.py --workload c4 --batch 1024 --steps 3 --no-cpu-baseline --inflight 1 > gpurun_out/b15_c4_$1.log 2>&1; show gpurun_out/b15_c4_$1.log c4_$1; done
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 3 -c 1 -o gpurun_out/r02d_tc_main python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "ncu main rc=$?"
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 2 -c 1 -o gpurun_out/r02d_tc_sample python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "ncu sample rc=$?"
