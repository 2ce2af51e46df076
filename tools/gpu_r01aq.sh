timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q -s > gpurun_out/pytest_aq.log 2>&1; echo pytest_rc=$?; grep -E "n=1024|n=2048|passed|failed|Error|assert" gpurun_out/pytest_aq.log | tail -8
for S in 7 6; do timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --slices $S --reps 2; done 2>&1 | tee gpurun_out/prof_aq.txt
timeout 600 python bench.py --root-precision auto6 --no-cpu-baseline > gpurun_out/bench_aq6.json 2> gpurun_out/bench_aq6.err; echo bench6_rc=$?; cut -c1-200 gpurun_out/bench_aq6.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 5 -c 1 -o gpurun_out/oz_gemm_tt_aq python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > gpurun_out/ncu_aq.log 2>&1; echo ncu=$?
