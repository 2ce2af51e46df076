#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh <tag>
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
timeout 300 tools/microbench/bin/ozaki_test > $O/ozaki_test.log 2>&1; echo "exit $?" >> $O/ozaki_test.log
if grep -q "^PASS" $O/ozaki_test.log; then
  SHAMPOO_OZAKI_PAIR=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_n1_pair.json 2> $O/bench_n1_pair.err
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_n1_single.json 2> $O/bench_n1_single.err
fi
echo done > $O/DONE
