#!/bin/bash
# Round evidence, run on the GPU box from the repo root:
#   bash profiles/collect.sh r02d
# -> gpurun_out/<tag>_tc_main.ncu-rep   ncu --set full of one K3 main launch (c3)
#    gpurun_out/<tag>_launches.csv      per-launch gpu__time_duration of c3 steps
#    gpurun_out/<tag>_bench_*.log       bench lines (ours for c1-c5, the reference arm for c3)
# Summarise here with profiles/summarize_ncu.py and profiles/launch_shares.py.
T=${1:-r02}
mkdir -p gpurun_out
# tensor-pipe issue rate of K3's MMA shapes in isolation (nvcc -O3 profiles/mma_rate.cu, built in the container)
[ -x profiles/mma_rate ] && ./profiles/mma_rate > gpurun_out/${T}_mma_rate.log 2>&1
# the 4th tc_score launch = the main pass of the 2nd run (each run: sample, main)
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 3 -c 1 -o gpurun_out/${T}_tc_main \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > gpurun_out/${T}_ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --inflight 1 > /dev/null 2>&1
python bench.py > gpurun_out/${T}_bench_c3.log 2>&1
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${T}_bench_c3_reference.log 2>&1
for w in "c1 --batch 1" "c2 --batch 1" "c2 --batch 256" "c3 --batch 1" "c4 --batch 1" "c4 --batch 1024 --steps 5" "c5 --batch 1 --k 1000" "c5 --batch 1 --k 1000 --low-pass"; do
  set -- $w
  python bench.py --workload $w --no-cpu-baseline > "gpurun_out/${T}_bench_$(echo $w | tr -d ' -').log" 2>&1
done
# tensor-heavy configs: one main K3 launch each (c2 B=256: run 1's main = the 4th tc_score launch;
# c4 B=1024: 4 sample + 4 main launches per run -> run 1's first main is the 13th)
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 3 -c 1 -o gpurun_out/${T}_tc_c2b256 \
  python bench.py --workload c2 --batch 256 --steps 1 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 12 -c 1 -o gpurun_out/${T}_tc_c4b1024 \
  python bench.py --workload c4 --batch 1024 --steps 1 --warmup 1 --no-cpu-baseline --inflight 1 > /dev/null 2>&1
