#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bench_path.py -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_smem.csv \
  python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > $O/launches_smem.log 2>&1
timeout 600 python tools/profile_root.py --batch 528 --hybrid -9 --reps 3 > $O/profile_smem.log 2>&1
cp paper_2002_09018_b200/libshampoo.so /tmp/lib_smem.so
cp tools/microbench/bin/libshampoo_mirror_shfl.so paper_2002_09018_b200/libshampoo.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_shfl.csv \
  python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > $O/launches_shfl.log 2>&1
timeout 600 python tools/profile_root.py --batch 528 --hybrid -9 --reps 3 > $O/profile_shfl.log 2>&1
cp /tmp/lib_smem.so paper_2002_09018_b200/libshampoo.so
timeout 600 python tools/profile_root.py --batch 528 --hybrid -9 --reps 3 > $O/profile_smem2.log 2>&1
echo done > $O/DONE
