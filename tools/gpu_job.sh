#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 300 tools/microbench/bin/ozaki_test > $O/ozaki_test.log 2>&1; echo "exit $?" >> $O/ozaki_test.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench_n1.json 2> $O/bench_n1.err
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_root528.csv \
  python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > $O/launches_root528.log 2>&1
echo done > $O/DONE
