timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_oz2.csv python tools/profile_root.py --batch 148 --reps 1 --hybrid -9 > /dev/null 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/launches_oz2.csv 2>/dev/null | head -6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 5 -c 1 -o gpurun_out/ozaki_gemm2 python tools/profile_root.py --batch 148 --reps 1 --hybrid -9 > /dev/null 2>&1; echo ncu_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:slice_kernel -s 5 -c 1 -o gpurun_out/ozaki_slice python tools/profile_root.py --batch 148 --reps 1 --hybrid -9 > /dev/null 2>&1; echo ncu_rc=$?
