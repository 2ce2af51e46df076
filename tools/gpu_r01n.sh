timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err; echo bench_rc=$?; cat gpurun_out/bench_n.json
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n.csv $CMD > /dev/null 2>&1; echo launch_rc=$?
python tools/launch_summary.py gpurun_out/launches_n.csv | head -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 0 -c 1 -o gpurun_out/tc_gemm_r01n python tools/profile_precondition.py --reps 1 > /dev/null 2>&1; echo ncu_tc_rc=$?
