timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
python tools/profile_precondition.py > gpurun_out/prof_prec.log 2>&1; cat gpurun_out/prof_prec.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prec.csv python tools/profile_precondition.py --reps 1 > /dev/null 2>&1; echo launch_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 0 -c 1 -o gpurun_out/tc_gemm_r01 python tools/profile_precondition.py --reps 1 > gpurun_out/ncu_tc.log 2>&1; echo ncu_rc=$?
