# final state: full GPU suite, smoke, N=1 bench (with cpu baseline), N=2/4 bench, multi-GPU bit identity
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_h.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_h.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_n1_h.json 2> gpurun_out/bench_n1_h.err; echo rc1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_h.json 2> gpurun_out/bench_n2_h.err; echo rc2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_n4_h.json 2> gpurun_out/bench_n4_h.err; echo rc4=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29583 tools/check_multi_gpu.py > gpurun_out/check_multi_h.log 2>&1; echo check_rc=$?; tail -2 gpurun_out/check_multi_h.log
grep -h metric gpurun_out/bench_n1_h.json gpurun_out/bench_n2_h.json gpurun_out/bench_n4_h.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], round(d['value'],1), round(d['ms_per_step'],1), d['phase_ms'], round(d['e2e']['value'],1), d['clocks'], round(d['roofline']['frac'],3) if d.get('roofline') else None)"
