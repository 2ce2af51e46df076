#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
rm -f tools/microbench/bin/ozaki_test   # the test must build it
timeout 1200 python -m pytest tests/test_gpu_ozaki_gemm.py -q -s > $O/pytest_gemm.log 2>&1; echo "pytest exit $?" >> $O/pytest_gemm.log
echo done > $O/DONE
