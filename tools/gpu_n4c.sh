# multi-GPU with the integer-epilogue Ozaki roots: N=4, N=2, N=1 back to back, and the bit-identity check
nvidia-smi -L
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_n4_w.json 2> gpurun_out/bench_n4_w.err; echo rc4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_w.json 2> gpurun_out/bench_n2_w.err; echo rc2=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_n1_w.json 2> gpurun_out/bench_n1_w.err; echo rc1=$?
timeout 600 python tools/check_multi_gpu.py > gpurun_out/check_multi_w.log 2>&1; echo check_rc=$?; tail -3 gpurun_out/check_multi_w.log
grep -h metric gpurun_out/bench_n1_w.json gpurun_out/bench_n2_w.json gpurun_out/bench_n4_w.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], round(d['value'],1), round(d['ms_per_step'],1), d['phase_ms'], d['clocks'])"
