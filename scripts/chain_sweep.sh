#!/bin/bash
# Tuning: k_rs_classify CTA size x shift CTAs per SM against the run time, default sum order.
cd "$GRAFT_REPO_ROOT" || exit 1
for ct in 256 128 64; do
for k in 6 7; do
  echo "classify threads $ct, shift CTAs per SM = $k"
  GRIDSHIFT_CLASSIFY_T=$ct GRIDSHIFT_SHIFT_CTAS=$k timeout 300 python scripts/prof_refsum.py 100000000 50 2>&1 | grep "^n="
done
done
