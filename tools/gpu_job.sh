#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
lscpu > $O/lscpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_path.py -q -rA -s > $O/pytest_bench_path.log 2>&1; echo "pytest exit $?" >> $O/pytest_bench_path.log
timeout 900 python tools/bench_delayed.py --chunks 32,16,8 > $O/delayed.json 2> $O/delayed.err
timeout 600 python tools/cpu_baseline.py > $O/cpu_baseline.json 2> $O/cpu_baseline.err
timeout 600 python tools/profile_stats.py --reps 3 > $O/stats_timing.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stats_kernel -s 1 -c 1 -f -o $O/stats \
  python tools/profile_stats.py --reps 2 > $O/ncu_stats.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/launches_step.log 2>&1
echo done > $O/DONE
