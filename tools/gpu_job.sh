#!/bin/bash
T=${1:-r02z}
O=gpurun_out/$T
mkdir -p $O
timeout 300 tools/microbench/bin/ozaki_test_pf > $O/pf.log 2>&1; echo "exit $?" >> $O/pf.log
timeout 300 tools/microbench/bin/ozaki_test > $O/full.log 2>&1; echo "exit $?" >> $O/full.log
timeout 300 tools/microbench/bin/ozaki_test_pf > $O/pf2.log 2>&1; echo "exit $?" >> $O/pf2.log
echo done > $O/DONE
