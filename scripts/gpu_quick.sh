#!/bin/bash
# Quick GPU check after a kernel change: gpu tests, plain bench, k_hist/k_shift launch times.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/q_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/q_pytest_gpu.log
timeout 600 python bench.py > $O/q_bench.json 2> $O/q_bench.err; echo "bench rc=$?" >> $O/q_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_hist|k_shift_tma" \
  --csv --log-file $O/q_hist.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/q_ncu.log 2>&1
tail -2 $O/q_pytest_gpu.log
