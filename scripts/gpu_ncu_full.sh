#!/bin/bash
# ncu --set full captures of selected kernels: KERNELS="name:skip name:skip ..."
# Keeps text summaries (details page) in gpurun_out/, the reports only if KEEP_REP=1.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
N=${NCU_N:-100000000}
IT=${NCU_IT:-50}
for ks in $KERNELS; do
  k=${ks%%:*}; skip=${ks##*:}
  tag=$(echo "${k}_$skip" | tr -c 'A-Za-z0-9_\n' '_')
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip $skip --launch-count 1 \
    -o /tmp/full_$tag python scripts/prof_refsum.py $N $IT > $O/full_$tag.log 2>&1
  echo "$k rc=$?"
  ncu -i /tmp/full_$tag.ncu-rep --page details --csv > $O/full_${tag}_details.csv 2>/dev/null
  ncu -i /tmp/full_$tag.ncu-rep --page source --csv --print-source sass > /tmp/src_$tag.csv 2>/dev/null
  head -c 3000000 /tmp/src_$tag.csv > $O/full_${tag}_source.csv
  [ -n "$KEEP_REP" ] && cp /tmp/full_$tag.ncu-rep $O/
done
du -sh $O
