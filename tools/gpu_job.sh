#!/bin/bash
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python bench.py --max-precond-dim 4096 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_config3p.json 2> $O/bench_config3p.err
bash tools/sweep_blocks.sh > $O/block_sweep.jsonl 2> $O/block_sweep.err
timeout 900 python tools/bench_workloads.py --workload config2 > $O/config2.json 2> $O/config2.err
timeout 900 python tools/bench_workloads.py --workload config4 > $O/config4.json 2> $O/config4.err
timeout 900 python tools/bench_workloads.py --workload resnet50 > $O/resnet50.json 2> $O/resnet50.err
echo done > $O/DONE
