#!/bin/bash
# K3 (c3 main pass) sensitivity sweep: one bench process per setting, prints
# the main-scorer launch time.  Diagnostics only (HYRE_TC_DEBUG runs return
# invalid results by design).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --inflight 1 ${BENCH_ARGS:-} \
    > gpurun_out/sweep.tmp 2> gpurun_out/sweep.err
  python - "$label" <<'PY'
import json, sys
try:
    l = [json.loads(x) for x in open("gpurun_out/sweep.tmp") if x.startswith("{")][-1]
    print(f"{sys.argv[1]:34s} main {l['stages_ms']['main_scorer']:.4f} ms  step {l['ms_per_step']:.4f}  frac {l['roofline']['frac']:.3f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/sweep.err").read()[-300:])
PY
}
for v in "$@"; do eval "run $v"; done
