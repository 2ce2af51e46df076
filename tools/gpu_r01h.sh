python tools/profile_stats.py > gpurun_out/prof_stats.log 2>&1; cat gpurun_out/prof_stats.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stats_kernel -s 2 -c 1 -o gpurun_out/stats_r01h python tools/profile_stats.py --reps 3 > gpurun_out/ncu_stats.log 2>&1; echo ncu_stats_rc=$?
python tools/profile_root.py --batch 148 > gpurun_out/prof_root.log 2>&1; cat gpurun_out/prof_root.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:root_kernel -s 1 -c 1 -o gpurun_out/root_r01h python tools/profile_root.py --batch 148 > gpurun_out/ncu_root.log 2>&1; echo ncu_root_rc=$?
timeout 600 python tools/bench_workloads.py --workload resnet50 > gpurun_out/wl_resnet50.json 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_resnet50.csv python tools/bench_workloads.py --workload resnet50 --steps 1 --warmup 1 > /dev/null 2>&1; echo launch_rc=$?
