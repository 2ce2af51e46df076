#!/bin/bash
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 300 tools/microbench/bin/ozaki_test_l2 > $O/l2.log 2>&1; echo "exit $?" >> $O/l2.log
timeout 300 tools/microbench/bin/ozaki_test > $O/full.log 2>&1; echo "exit $?" >> $O/full.log
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:gemm -c 9 --csv tools/microbench/bin/ozaki_test > $O/ncu_full.csv 2>&1
echo done > $O/DONE
