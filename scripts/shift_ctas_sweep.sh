#!/bin/bash
# Tuning: persistent shift CTAs per SM (GRIDSHIFT_SHIFT_CTAS) against the run time, default sum order.
cd "$GRAFT_REPO_ROOT" || exit 1
for k in 8 7 6 5 4 3; do
  echo "shift CTAs per SM = $k"
  GRIDSHIFT_SHIFT_CTAS=$k timeout 300 python scripts/prof_refsum.py 100000000 50 2>&1 | grep "^n="
done
