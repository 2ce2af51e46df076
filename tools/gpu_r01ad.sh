# full GPU suite + default bench (prefetching e2e) + launch list of the bench step + ncu --set full of a GEMM
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ad.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_ad.log
timeout 600 python bench.py > gpurun_out/bench_ad.json 2> gpurun_out/bench_ad.err; echo bench_rc=$?; cat gpurun_out/bench_ad.json; tail -3 gpurun_out/bench_ad.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ad.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ad.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/oz_gemm_ad python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > gpurun_out/ncu_ad2.log 2>&1; echo ncu2=$?
