#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 600 tools/microbench/bin/slice_layout 528 > $O/slice_layout.log 2>&1; echo "exit $?" >> $O/slice_layout.log
echo done > $O/DONE
