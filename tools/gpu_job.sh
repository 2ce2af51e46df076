#!/bin/bash
# One gpurun session (round 2).  gpurun --timeout 2700 -- bash tools/gpu_job.sh r02b
T=${1:-r02x}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bench_path.py -q -rA -s > $O/pytest_bench_path.log 2>&1; echo "pytest exit $?" >> $O/pytest_bench_path.log
timeout 900 python tools/check_concurrency.py > $O/concurrency.jsonl 2> $O/concurrency.err; echo "exit $?" >> $O/concurrency.err
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_small.py > $O/memcheck.log 2>&1; echo "exit $?" >> $O/memcheck.log
echo done > $O/DONE
