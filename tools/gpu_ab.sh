for i in 1 2; do
  (cd abtest/old && python tools/profile_root.py --batch 296 --reps 2 && python tools/profile_stats.py --reps 3) 2>&1 | grep -E "roots/s|stats:" | sed "s/^/old: /"
  (python tools/profile_root.py --batch 296 --reps 2 && python tools/profile_stats.py --reps 3) 2>&1 | grep -E "roots/s|stats:" | sed 's/^/new: /'
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
