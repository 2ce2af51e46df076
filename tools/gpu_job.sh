#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
timeout 300 tools/microbench/bin/ozaki_test > $O/ozaki_test.log 2>&1; echo "exit $?" >> $O/ozaki_test.log
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bench_path.py tests/test_gpu_parity.py -q -rA -s > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_n1.json 2> $O/bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_root528.csv \
  python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > $O/launches_root528.log 2>&1
echo done > $O/DONE
