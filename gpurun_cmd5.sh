set -u
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest5.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/gputest5.log
ncu --set full --clock-control none --import-source on -k regex:tc_score -s 3 -c 1 -o gpurun_out/r02b_tc_main \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --inflight 1 > gpurun_out/r02b_ncu_full.log 2>&1; echo "ncu rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02b_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --inflight 1 > /dev/null 2>&1; echo "launches rc=$?"
