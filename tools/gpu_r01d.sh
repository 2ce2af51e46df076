# round-1 re-entry: parity, bench N=1, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_d.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_d.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke_d.log
timeout 600 python bench.py > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo bench_rc=$?
cat gpurun_out/bench_d.json
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_d.csv $CMD > gpurun_out/ncu_launch_d.log 2>&1; echo launch_rc=$?
