for w in config2 config4 resnet50; do
  timeout 600 python tools/bench_workloads.py --workload $w > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err; echo "$w rc=$?"; cat gpurun_out/wl_$w.json; tail -3 gpurun_out/wl_$w.err
done
