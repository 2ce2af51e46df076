mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_e.log 2>&1; echo pytest_rc=$?; tail -30 gpurun_out/pytest_gpu_e.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo bench_rc=$?; cat gpurun_out/bench_e.json
