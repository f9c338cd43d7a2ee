#!/bin/bash
# One GPU session: gpu tests, plain bench, launch list, traffic pass, full capture.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_shift_tma|k_hist" \
  --csv --log-file $O/traffic.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_shift|k_agg_brick3|k_derive_brick3|k_bk_|k_init_aos|k_hist" -c 10 \
  -o $O/full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1

# keep the copy-back under gpurun's 64 MiB cap
ncu -i $O/full.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
ncu -i $O/full.ncu-rep --page details --csv > $O/full_details.csv 2>/dev/null
gzip -f $O/launches.csv $O/full_raw.csv $O/full_details.csv $O/traffic.csv 2>/dev/null
sz=$(du -sm $O | cut -f1); if [ "$sz" -gt 60 ]; then rm -f $O/full.ncu-rep; fi
du -sh $O/*
