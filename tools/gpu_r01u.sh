# round-1 re-entry check: full GPU suite + default bench on the committed state
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_u.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_u.log
timeout 600 python bench.py > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err; echo bench_rc=$?; cat gpurun_out/bench_u.json
