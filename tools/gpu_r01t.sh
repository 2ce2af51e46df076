timeout 600 python bench.py > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err; echo bench_rc=$?; cat gpurun_out/bench_t.json
timeout 600 python tools/bench_workloads.py --workload config2 > gpurun_out/wl_config2_oz.json 2>&1; tail -1 gpurun_out/wl_config2_oz.json
timeout 600 python tools/bench_workloads.py --workload resnet50 > gpurun_out/wl_resnet50_oz.json 2>&1; tail -1 gpurun_out/wl_resnet50_oz.json
timeout 600 python tools/bench_workloads.py --workload config4 > gpurun_out/wl_config4_oz.json 2>&1; tail -1 gpurun_out/wl_config4_oz.json
