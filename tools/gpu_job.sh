#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python tools/profile_layer_ranks.py --world 1 2 4 8 --owners tensor root > $O/layer_ranks.jsonl 2> $O/layer_ranks.err
for w in config2 config4 resnet50; do timeout 900 python tools/bench_workloads.py --workload $w > $O/workload_$w.json 2> $O/workload_$w.err; done
echo done > $O/DONE
