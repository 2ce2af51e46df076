# root exchange: overlapped per-group broadcasts vs one all-gather, N=2 and N=4
for N in 4 2; do for G in overlapped allgather; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 3 --warmup 3 --gather $G --no-cpu-baseline > gpurun_out/bench_n${N}_g_$G.json 2> gpurun_out/bench_n${N}_g_$G.err; echo N=$N $G rc=$?
done; done
for f in gpurun_out/bench_n4_g_overlapped.json gpurun_out/bench_n4_g_allgather.json gpurun_out/bench_n2_g_overlapped.json gpurun_out/bench_n2_g_allgather.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['value'],1), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['phase_ms'].items()}, round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"; done
