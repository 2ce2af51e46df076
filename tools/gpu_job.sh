#!/bin/bash
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 600 python tools/debug_err_history.py 24 > $O/err.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bench_path.py -q > $O/pytest_oz.log 2>&1; echo "pytest exit $?" >> $O/pytest_oz.log
timeout 600 python tools/profile_root.py --batch 528 --hybrid -9 --reps 2 > $O/profile_root.log 2>&1
SHAMPOO_OZAKI_DUAL=0 timeout 600 python tools/profile_root.py --batch 528 --hybrid -9 --reps 2 >> $O/profile_root.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_root528.csv \
  python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > $O/launches_root528.log 2>&1
echo done > $O/DONE
