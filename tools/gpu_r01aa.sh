# register slicing incl. T-from-M, pinned fp64 conversions, integer abs: tests, timing, launch list, bench
timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q -s > gpurun_out/pytest_oz_aa.log 2>&1; echo pytest_rc=$?; grep -E "n=1024|passed|failed|Error" gpurun_out/pytest_oz_aa.log | tail -8
for S in 7 6; do timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --slices $S --reps 2; done 2>&1 | tee gpurun_out/prof_aa.txt
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_kernel|slice" -c 14 --csv --log-file gpurun_out/launches_aa.csv python tools/profile_root.py --batch 528 --hybrid -9 --slices 7 --reps 1 > gpurun_out/ncu_aa.log 2>&1; echo ncu_rc=$?
timeout 600 python bench.py > gpurun_out/bench_aa.json 2> gpurun_out/bench_aa.err; echo bench_rc=$?; cat gpurun_out/bench_aa.json
