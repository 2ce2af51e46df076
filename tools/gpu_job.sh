#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
timeout 900 tools/microbench/bin/ozaki_test > $O/ozaki_test.log 2>&1; echo "exit $?" >> $O/ozaki_test.log
echo done > $O/DONE
