#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
for P in stages2 stages3 stagesmax; do timeout 300 tools/microbench/bin/oz_$P > $O/oz_$P.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -rA -s -k "tail or 2048 or 1024" > $O/pytest_ozaki.log 2>&1; echo "pytest exit $?" >> $O/pytest_ozaki.log
echo done > $O/DONE
