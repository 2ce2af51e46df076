# BK 32 vs 64 (microbench + real root), ncu --set full of the P1 GEMM
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -I paper_2002_09018_b200/csrc tools/microbench/ozaki_test.cu -lcuda -o /tmp/ozaki_test && timeout 300 /tmp/ozaki_test > gpurun_out/ozaki_test_ab.txt 2>&1; echo micro_rc=$?; grep "1024\|PASS\|FAIL" gpurun_out/ozaki_test_ab.txt
for bk in 64 32 64 32; do SHAMPOO_OZ_BK=$bk timeout 300 python tools/profile_root.py --batch 528 --hybrid -9 --slices 7 --reps 2 | sed "s/^/BK=$bk /"; done 2>&1 | tee gpurun_out/prof_ab.txt
SHAMPOO_OZ_BK=32 timeout 900 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/pytest_oz_ab.log 2>&1; echo pytest32_rc=$?; tail -1 gpurun_out/pytest_oz_ab.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/oz_gemm_p1_ab python tools/profile_root.py --batch 528 --hybrid -9 --reps 1 > gpurun_out/ncu_ab.log 2>&1; echo ncu=$?
