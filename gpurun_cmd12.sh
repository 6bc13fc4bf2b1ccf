set -u
mkdir -p gpurun_out
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; }
HYRE_TC_BIAS=0 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b12_c4_nobias.log 2>&1; show gpurun_out/b12_c4_nobias.log c4_nobias
HYRE_TC_BIAS=0 HYRE_TC_DEBUG=2 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b12_c4_nobias_noepi.log 2>&1; show gpurun_out/b12_c4_nobias_noepi.log c4_nobias_noepi
HYRE_TC_SAMPLE_SEGS=60 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b12_c4_s60.log 2>&1; show gpurun_out/b12_c4_s60.log c4_segs60
HYRE_TC_BIAS=0 timeout 600 python bench.py --workload c2 --batch 256 --no-cpu-baseline --inflight 1 > gpurun_out/b12_c2_nobias.log 2>&1; show gpurun_out/b12_c2_nobias.log c2B256_nobias
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 12 -c 1 -o gpurun_out/r02_tc_c4b1024_main python bench.py --workload c4 --batch 1024 --steps 1 --warmup 1 --no-cpu-baseline --inflight 1 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
