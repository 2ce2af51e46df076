timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q -s -k "bound or 2048" > gpurun_out/pytest_as.log 2>&1; echo pytest_rc=$?; tail -25 gpurun_out/pytest_as.log
