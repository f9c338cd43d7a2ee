#!/bin/bash
# GPU check: full gpu test suite (incl. slow), then a short bench.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > $O/c_pytest.log 2>&1; echo "pytest rc=$?" >> $O/c_pytest.log
tail -40 $O/c_pytest.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/c_bench.json 2> $O/c_bench.err; echo "bench rc=$?" >> $O/c_bench.err
tail -3 $O/c_bench.err
fi
