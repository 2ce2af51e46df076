# power iteration with integer-pipe fp32->fp64 widening (XU pipe was saturated)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_av.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_av.log
timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --slices 7 --reps 2 2>&1 | tee gpurun_out/prof_av.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -k regex:"root_kernel" -c 1 --csv --log-file gpurun_out/launches_av.csv python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > gpurun_out/ncu_av.log 2>&1; echo ncu_rc=$?
timeout 600 python tools/bench_workloads.py --workload config2 > gpurun_out/wl_config2_av.json 2>&1; tail -1 gpurun_out/wl_config2_av.json | cut -c1-300
timeout 600 python bench.py > gpurun_out/bench_av.json 2> gpurun_out/bench_av.err; echo bench_rc=$?; cut -c1-250 gpurun_out/bench_av.json
