#!/bin/bash
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_bench.log 2>&1
echo done > $O/DONE
