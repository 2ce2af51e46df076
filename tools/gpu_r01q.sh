timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench_rc=$?; cat gpurun_out/bench_q.json
timeout 600 python bench.py --root-precision fp64 --no-cpu-baseline > gpurun_out/bench_q_fp64.json 2> gpurun_out/bench_q_fp64.err; echo bench_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv $CMD > /dev/null 2>&1; echo launch_rc=$?
python tools/launch_summary.py gpurun_out/launches_q.csv > gpurun_out/launches_q.txt 2>&1; head -12 gpurun_out/launches_q.txt
