set -u
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest10.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest10.log
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()}, 'e2e', round(d.get('e2e',{}).get('value',0)))"; }
timeout 600 python bench.py --workload c1 --batch 1 --no-cpu-baseline > gpurun_out/b10_c1.log 2>&1; show gpurun_out/b10_c1.log c1
timeout 600 python bench.py --workload c2 --batch 256 --no-cpu-baseline > gpurun_out/b10_c2_256.log 2>&1; show gpurun_out/b10_c2_256.log c2B256
timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline > gpurun_out/b10_c4_1024.log 2>&1; show gpurun_out/b10_c4_1024.log c4B1024
HYRE_TC_DEBUG=128 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b10_c4_tmem.log 2>&1; show gpurun_out/b10_c4_tmem.log c4B1024_tmemonly
HYRE_TC_DEBUG=2 timeout 900 python bench.py --workload c4 --batch 1024 --steps 5 --no-cpu-baseline --inflight 1 > gpurun_out/b10_c4_noepi.log 2>&1; show gpurun_out/b10_c4_noepi.log c4B1024_noepi
ncu --set full --clock-control none --import-source on -k regex:select_prefilter -s 2 -c 1 -o gpurun_out/r02_k4p python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "ncu k4p rc=$?"
