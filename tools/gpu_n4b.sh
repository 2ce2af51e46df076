timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_n4_oz.json 2> gpurun_out/bench_n4_oz.err; echo rc4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_oz.json 2> gpurun_out/bench_n2_oz.err; echo rc2=$?
grep -h metric gpurun_out/bench_n4_oz.json gpurun_out/bench_n2_oz.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], round(d['value'],1), round(d['ms_per_step'],1), d['phase_ms'], d['clocks'])"
