# cluster power iteration (lambda_hat from shared-memory-resident matrices)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ae.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_ae.log
timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --slices 7 --reps 2 2>&1 | tee gpurun_out/prof_ae.txt
timeout 300 python tools/profile_root.py --batch 528 --reps 2 --max-iter 0 2>&1 | tee -a gpurun_out/prof_ae.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pi_cluster|root_kernel" -c 4 --csv --log-file gpurun_out/launches_ae.csv python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > gpurun_out/ncu_ae.log 2>&1; echo ncu_rc=$?
timeout 600 python bench.py > gpurun_out/bench_ae.json 2> gpurun_out/bench_ae.err; echo bench_rc=$?; cat gpurun_out/bench_ae.json
timeout 600 python tools/bench_workloads.py --workload config2 > gpurun_out/wl_config2_ae.json 2>&1; tail -1 gpurun_out/wl_config2_ae.json
