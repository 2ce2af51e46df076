python tests/evidence/hybrid_switch.py 2>&1 | tail -6
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hybrid2.csv python tools/profile_root.py --batch 148 --reps 1 --hybrid 8 > /dev/null 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/launches_hybrid2.csv | head -4
