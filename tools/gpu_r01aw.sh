# Ozaki-path root_kernel<true> (no DMMA code: 4 CTAs/SM for the power sweeps)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_aw.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_aw.log
timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --slices 7 --reps 2 2>&1 | tee gpurun_out/prof_aw.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"root_kernel" -c 1 --csv --log-file gpurun_out/launches_aw.csv python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > gpurun_out/ncu_aw.log 2>&1; echo ncu_rc=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_aw.json 2> gpurun_out/bench_aw.err; echo bench_rc=$?; cut -c1-250 gpurun_out/bench_aw.json; grep -o '"phase_ms": {[^}]*}' gpurun_out/bench_aw.json; grep -o '"root_kernel_ms_power_iteration_and_setup": [0-9.]*' gpurun_out/bench_aw.json
