#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
timeout 300 tools/microbench/bin/ozaki_test_epi16 > $O/ozaki_test_epi16.log 2>&1; echo "exit $?" >> $O/ozaki_test_epi16.log
timeout 300 tools/microbench/bin/oz_probe0 > $O/oz_epi8.log 2>&1
timeout 300 tools/microbench/bin/oz_epi16 > $O/oz_epi16.log 2>&1
timeout 300 tools/microbench/bin/oz_probe0 > $O/oz_epi8b.log 2>&1
echo done > $O/DONE
