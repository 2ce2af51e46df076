#!/bin/bash
# One gpurun session (round 2): GPU tests, smoke, bench, f1 measurement, ncu launch list + full capture.
#   gpurun --timeout 2700 -- bash tools/gpu_job.sh r02a
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 python tools/bench_delayed.py > $O/delayed.json 2> $O/delayed.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_root528.csv \
  python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > $O/launches_root528.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 8 -c 4 -f -o $O/gemm148 \
  python tools/profile_root.py --batch 148 --hybrid -9 --reps 1 > $O/ncu_gemm148.log 2>&1
echo done > $O/DONE
