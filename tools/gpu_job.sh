#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:"slice|root_kernel" -c 4 -f -o $O/slices148 \
  python tools/profile_root.py --batch 148 --hybrid -9 --reps 1 > $O/ncu_slices148.log 2>&1
echo done > $O/DONE
