set -u
mkdir -p gpurun_out
T=r02
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 3 -c 1 -o gpurun_out/${T}_tc_main \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu c3 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:tc_score|hist_thr|select|run_init' -s 10 -c 10 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 1 -c 2 -o gpurun_out/${T}_tc_c2b256 \
  python bench.py --workload c2 --batch 256 --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > gpurun_out/${T}_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 4 -c 2 -o gpurun_out/${T}_tc_c4b1024 \
  python bench.py --workload c4 --batch 1024 --steps 1 --warmup 0 --no-cpu-baseline --inflight 1 > gpurun_out/${T}_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
bash profiles/sanitize.sh
