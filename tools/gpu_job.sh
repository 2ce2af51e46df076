#!/bin/bash
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
for g in 0 8 16 24 36; do
  SHAMPOO_PI_GROUP=$g timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --reps 2 --digest >> $O/pi_group.log 2>&1
  SHAMPOO_PI_GROUP=$g timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:root_kernel \
     --log-file $O/pi_group_$g.csv python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > /dev/null 2>&1
done
timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --reps 2 --digest >> $O/pi_group.log 2>&1
echo done > $O/DONE
