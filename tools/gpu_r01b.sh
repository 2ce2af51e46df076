set -x
timeout 600 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; echo bench_rc=$?
cat gpurun_out/bench_r01b.json
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_short.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"root_kernel|stats_kernel|check_kernel|prep_kernel|diag_kernel|finish_kernel|prec_" --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
python tools/profile_root.py --batch 148 > gpurun_out/prof_root_plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:root_kernel -s 1 -c 1 -o gpurun_out/root_r01b python tools/profile_root.py --batch 148 > gpurun_out/ncu_root2.log 2>&1; echo ncu_rc=$?
