#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r100_launches.csv python scripts/prof_refsum.py 100000000 50 > $O/r100_ncu.log 2>&1
echo "ncu rc=$?"
tail -2 $O/r100_ncu.log
