#!/bin/bash
# Tuning: shift CTAs per SM (GRIDSHIFT_SHIFT_CTAS; <= 8 resident: persistent, more: several waves) and
# the table chain's stream priority (GRIDSHIFT_SIDE_PRIO) against the run time, default sum order.
cd "$GRAFT_REPO_ROOT" || exit 1
for pr in low high; do
for k in ${SWEEP:-6 8 16 32 64 128}; do
  echo "side priority $pr, shift CTAs per SM = $k"
  GRIDSHIFT_SIDE_PRIO=$pr GRIDSHIFT_SHIFT_CTAS=$k timeout 300 python scripts/prof_refsum.py 100000000 50 2>&1 | grep "^n="
done
done
