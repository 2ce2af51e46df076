# A/B of the root kernel variants on one box + rational parity
for i in 1 2; do
  (cd abtest/old && python tools/profile_root.py --batch 296 --reps 3) 2>&1 | tail -1 | sed "s/^/old: /"
  python tools/profile_root.py --batch 296 --reps 3 2>&1 | tail -1 | sed 's/^/new: /'
done
python tools/profile_root.py --batch 148 --reps 2 --p 8 2>&1 | tail -1 | sed 's/^/new p8: /'
python tools/profile_root.py --batch 148 --reps 2 --p 6 2>&1 | tail -1 | sed 's/^/new p6: /'
timeout 600 python -m pytest tests/test_gpu_rational.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
