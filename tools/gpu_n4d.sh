# final-state numbers: smoke, secondary workloads, N=1/2/4 bench, multi-GPU bit identity
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python tools/bench_workloads.py --workload config2 > gpurun_out/wl_config2_z.json 2>&1; tail -1 gpurun_out/wl_config2_z.json | cut -c1-400
timeout 600 python tools/bench_workloads.py --workload config4 > gpurun_out/wl_config4_z.json 2>&1; tail -1 gpurun_out/wl_config4_z.json | cut -c1-400
timeout 600 python tools/bench_workloads.py --workload resnet50 > gpurun_out/wl_resnet50_z.json 2>&1; tail -1 gpurun_out/wl_resnet50_z.json | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_n4_z.json 2> gpurun_out/bench_n4_z.err; echo rc4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_z.json 2> gpurun_out/bench_n2_z.err; echo rc2=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_n1_z.json 2> gpurun_out/bench_n1_z.err; echo rc1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 tools/check_multi_gpu.py > gpurun_out/check_multi_z.log 2>&1; echo check_rc=$?; tail -3 gpurun_out/check_multi_z.log
grep -h metric gpurun_out/bench_n1_z.json gpurun_out/bench_n2_z.json gpurun_out/bench_n4_z.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], round(d['value'],1), round(d['ms_per_step'],1), d['phase_ms'], d['e2e']['value'], d['clocks'])"
