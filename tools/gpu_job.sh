#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python tools/check_group_streams.py --reps 3 > $O/group_streams.json 2> $O/group_streams.err
echo done > $O/DONE
