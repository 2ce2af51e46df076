for i in 1 2; do
  (cd abtest/old && python tools/profile_stats.py --reps 5) 2>&1 | tail -1 | sed "s/^/old: /"
  python tools/profile_stats.py --reps 5 2>&1 | tail -1 | sed 's/^/new: /'
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stats" 2>&1 | tail -2
