# integer epilogue + register-cached slicing + S = 6 option: microbench, Ozaki tests, root timing, bench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -I paper_2002_09018_b200/csrc tools/microbench/ozaki_test.cu -lcuda -o /tmp/ozaki_test && timeout 300 /tmp/ozaki_test > gpurun_out/ozaki_test_w.txt 2>&1; echo micro_rc=$?; cat gpurun_out/ozaki_test_w.txt
timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q -s > gpurun_out/pytest_oz_w.log 2>&1; echo pytest_rc=$?; grep -E "n=1024|passed|failed|Error" gpurun_out/pytest_oz_w.log | tail -8
for S in 7 6; do timeout 300 python tools/profile_root.py --batch 148 --hybrid -9 --slices $S --reps 2; done 2>&1 | tee gpurun_out/prof_w.txt
timeout 600 python bench.py > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err; echo bench_rc=$?; cat gpurun_out/bench_w.json
timeout 600 python bench.py --root-precision auto6 --no-cpu-baseline > gpurun_out/bench_w6.json 2> gpurun_out/bench_w6.err; echo bench6_rc=$?; cat gpurun_out/bench_w6.json
