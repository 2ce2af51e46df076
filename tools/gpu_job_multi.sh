#!/bin/bash
# Multi-GPU session (round 2): gpurun --gpus N --timeout 2400 -- bash tools/gpu_job_multi.sh <tag> N [tests]
T=${1:-r02m}
N=${2:-2}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
if [ "$3" == "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rA -s > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
fi
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $R tools/check_multi_gpu.py --full --shard layers > $O/check_layers_n$N.txt 2>&1; echo "exit $?" >> $O/check_layers_n$N.txt
timeout 600 $R tools/check_multi_gpu.py --shard roots > $O/check_roots_n$N.txt 2>&1; echo "exit $?" >> $O/check_roots_n$N.txt
timeout 600 $R tools/check_delayed_multi.py > $O/check_delayed_n$N.txt 2>&1; echo "exit $?" >> $O/check_delayed_n$N.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 $R bench.py --gpus $N --steps 5 --warmup 3 --shard layers > $O/bench_n${N}_layers.json 2> $O/bench_n${N}_layers.err
timeout 900 $R bench.py --gpus $N --steps 5 --warmup 3 --shard roots > $O/bench_n${N}_roots.json 2> $O/bench_n${N}_roots.err
echo done > $O/DONE
