python tools/debug_hybrid.py 2>&1 | tail -12
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hybrid.csv python tools/profile_root.py --batch 148 --reps 1 --hybrid -1 > /dev/null 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/launches_hybrid.csv
