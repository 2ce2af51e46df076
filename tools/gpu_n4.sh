nvidia-smi -L
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo rc=$?; grep metric gpurun_out/bench_n4.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/check_multi_gpu.py > gpurun_out/check_multi4.log 2>&1; echo check_rc=$?; tail -3 gpurun_out/check_multi4.log
