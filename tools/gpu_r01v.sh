# ncu --set full of the current Ozaki GEMM and slice kernels (one 148-matrix root call)
timeout 300 python tools/profile_root.py --batch 148 --hybrid -9 --reps 1 > gpurun_out/prof_v_plain.txt 2>&1; cat gpurun_out/prof_v_plain.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 -o gpurun_out/oz_gemm_v python tools/profile_root.py --batch 148 --hybrid -9 --reps 1 > gpurun_out/ncu_v_gemm.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slice_kernel -s 6 -c 1 -o gpurun_out/oz_slice_v python tools/profile_root.py --batch 148 --hybrid -9 --reps 1 > gpurun_out/ncu_v_slice.log 2>&1; echo ncu2=$?
