set -u
mkdir -p gpurun_out
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; }
HYRE_TC_BACKOFF_NS=0 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b11_c4_bo0.log 2>&1; show gpurun_out/b11_c4_bo0.log c4_bo0
HYRE_TC_BACKOFF_NS=0 HYRE_TC_DEBUG=2 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b11_c4_bo0_noepi.log 2>&1; show gpurun_out/b11_c4_bo0_noepi.log c4_bo0_noepi
HYRE_TC_DEBUG=3 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b11_c4_nomma.log 2>&1; show gpurun_out/b11_c4_nomma.log c4_nomma_noepi
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 9 -c 1 -o gpurun_out/r02_tc_c4b1024 python bench.py --workload c4 --batch 1024 --steps 1 --warmup 1 --no-cpu-baseline --inflight 1 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 3 -c 1 -o gpurun_out/r02_tc_c2b256 python bench.py --workload c2 --batch 256 --steps 1 --warmup 1 --no-cpu-baseline --inflight 1 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
