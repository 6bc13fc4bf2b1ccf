set -u
mkdir -p gpurun_out
show() { grep '^{' "$1" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['p50_ms'], {k: round(v,4) for k,v in d['stages_ms'].items()})"; }
for s in 60 90 120 160 200 240 60; do HYRE_TC_SAMPLE_SEGS=$s timeout 600 python bench.py --no-cpu-baseline --inflight 1 > gpurun_out/b20_s$s.log 2>&1; show gpurun_out/b20_s$s.log segs$s; done
