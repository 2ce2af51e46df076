#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
for P in 0 1 2 3; do timeout 300 tools/microbench/bin/oz_probe$P > $O/oz_probe$P.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_bench_path.py -q -rA -s > $O/pytest_bench_path.log 2>&1; echo "pytest exit $?" >> $O/pytest_bench_path.log
echo done > $O/DONE
