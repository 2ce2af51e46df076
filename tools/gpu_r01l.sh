timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; echo rc=$?; cat gpurun_out/bench_l.json
timeout 600 python bench.py --steps 3 --warmup 3 --hybrid --no-cpu-baseline > gpurun_out/bench_l_hybrid.json 2> gpurun_out/bench_l_hybrid.err; echo rc=$?; cat gpurun_out/bench_l_hybrid.json
