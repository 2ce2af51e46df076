#!/bin/bash
# Final validation on a 4-GPU box (round 2): gpurun --gpus 4 --timeout 3000 -- bash tools/gpu_job_final.sh <tag>
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA -s > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
timeout 600 $R4 tools/check_multi_gpu.py --full --shard layers > $O/check_layers_n4.txt 2>&1; echo "exit $?" >> $O/check_layers_n4.txt
timeout 600 $R4 tools/check_multi_gpu.py --shard roots > $O/check_roots_n4.txt 2>&1; echo "exit $?" >> $O/check_roots_n4.txt
timeout 600 $R4 tools/check_delayed_multi.py > $O/check_delayed_n4.txt 2>&1; echo "exit $?" >> $O/check_delayed_n4.txt
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 $R2 bench.py --gpus 2 --steps 5 --warmup 3 --shard layers > $O/bench_n2_layers.json 2> $O/bench_n2_layers.err
timeout 900 $R4 bench.py --gpus 4 --steps 5 --warmup 3 --shard layers > $O/bench_n4_layers.json 2> $O/bench_n4_layers.err
timeout 900 $R4 bench.py --gpus 4 --steps 5 --warmup 3 --shard roots > $O/bench_n4_roots.json 2> $O/bench_n4_roots.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python tools/bench_delayed.py --chunks 32,16 > $O/delayed.json 2> $O/delayed.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_root528.csv \
  python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > $O/launches_root528.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 48 -c 4 -f -o $O/gemm148 \
  python tools/profile_root.py --batch 148 --hybrid -9 --reps 1 > $O/ncu_gemm148.log 2>&1
echo done > $O/DONE
