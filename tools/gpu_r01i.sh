timeout 600 python -m pytest tests/test_gpu_hybrid.py -q -x 2>&1 | tail -30
python tools/profile_root.py --batch 296 --reps 2 2>&1 | tail -1
python tools/profile_root.py --batch 296 --reps 2 --hybrid -1 2>&1 | tail -3
