set -u
mkdir -p gpurun_out
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; }
for s in 100 150 300; do HYRE_TC_SAMPLE_SEGS=$s timeout 900 python bench.py --workload c4 --batch 1024 --steps 3 --no-cpu-baseline --inflight 1 > gpurun_out/b25_c4_s$s.log 2>&1; show gpurun_out/b25_c4_s$s.log c4_segs$s; done
for s in 8 15 30; do HYRE_TC_SAMPLE_SEGS=$s timeout 900 python bench.py --workload c2 --batch 256 --no-cpu-baseline --inflight 1 > gpurun_out/b25_c2_s$s.log 2>&1; show gpurun_out/b25_c2_s$s.log c2_segs$s; done
ncu --set full --clock-control none --import-source on -k regex:select_prefilter -s 2 -c 1 -o gpurun_out/r02g_k4p python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "ncu k4p rc=$?"
