# T^m sliced in the GEMM epilogue (whole-sector row stores + warp-transposed mirror): tests, timing, launches, bench
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_ao.log 2>&1; echo pytest_rc=$?; grep -E "n=1024|n=2048|passed|failed|Error|assert" gpurun_out/pytest_ao.log | tail -8
timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --slices 7 --reps 2 2>&1 | tee gpurun_out/prof_ao.txt
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_kernel|slice" -c 8 --csv --log-file gpurun_out/launches_ao.csv python tools/profile_root.py --batch 528 --hybrid -9 --slices 7 --reps 1 > gpurun_out/ncu_ao.log 2>&1; echo ncu_rc=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ao.json 2> gpurun_out/bench_ao.err; echo bench_rc=$?; cat gpurun_out/bench_ao.json; tail -2 gpurun_out/bench_ao.err
