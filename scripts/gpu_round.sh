#!/bin/bash
# One GPU session: gpu tests, plain bench (cfg4) + reference arm + cfg2 leg, per-configuration timings,
# launch lists, traffic pass, full captures.  Outputs in gpurun_out/.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --workload cfg2 --steps 5 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python scripts/bench_configs.py cfg0 cfg1 cfg2 cfg3 cfg4 > $O/configs.json 2> $O/configs.err
timeout 900 python scripts/sum_modes_check.py > $O/sum_modes.json 2> $O/sum_modes.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_shift_tma|k_hist" \
  --csv --log-file $O/traffic.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_traffic.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/cfg2_launches.csv python bench.py --workload cfg2 --steps 1 --warmup 3 > $O/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_shift|k_agg_brick3|k_derive_brick3|k_rs_classify|k_rs_runfold|k_bk_|k_init_aos|k_hist" -c 14 \
  -o $O/full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1

# keep the copy-back under gpurun's 64 MiB cap
ncu -i $O/full.ncu-rep --page raw --csv > $O/full_raw.csv 2>/dev/null
ncu -i $O/full.ncu-rep --page details --csv > $O/full_details.csv 2>/dev/null
gzip -f $O/launches.csv $O/full_raw.csv $O/full_details.csv $O/traffic.csv $O/cfg2_launches.csv 2>/dev/null
sz=$(du -sm $O | cut -f1); if [ "$sz" -gt 60 ]; then rm -f $O/full.ncu-rep; fi
du -sh $O/*
