#!/bin/bash
# Reference-order sums: parity subset, run timings (reference vs exact order), launch list.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${PYTEST_K:-cfg4 or step_vs_reference or trajectory or reference_suite or tables_vs}" > $O/r_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r_pytest.log
tail -5 $O/r_pytest.log
for m in ref exact; do timeout 600 python scripts/prof_refsum.py 100000000 50 $m >> $O/r_time.log 2>&1; done
timeout 600 python scripts/prof_refsum.py 10000000 50 >> $O/r_time.log 2>&1
cat $O/r_time.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r_launches.csv python scripts/prof_refsum.py ${NCU_N:-100000000} ${NCU_IT:-50} > $O/r_ncu.log 2>&1
echo "ncu rc=$?"
