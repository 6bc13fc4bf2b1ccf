set -u
mkdir -p gpurun_out
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; }
for g in 296 148 74 37; do HYRE_TC_SAMPLE_GRID=$g timeout 600 python bench.py --no-cpu-baseline --inflight 1 --steps 30 > gpurun_out/b19_g$g.log 2>&1; show gpurun_out/b19_g$g.log grid$g; done
for s in 30 60 120; do HYRE_TC_SAMPLE_SEGS=$s timeout 600 python bench.py --no-cpu-baseline --inflight 1 --steps 30 > gpurun_out/b19_s$s.log 2>&1; show gpurun_out/b19_s$s.log segs$s; done
