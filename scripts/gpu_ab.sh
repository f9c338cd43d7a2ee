#!/bin/bash
# A/B timing: default library vs variants/lib_*.so, interleaved, 3 rounds.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
for r in 1 2 3; do
for lib in paper_2104_00303_b200/libgridshift_cuda.so variants/lib_*.so; do
  name=$(basename $lib .so)
  GRIDSHIFT_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/ab_${name}_$r.json 2>/dev/null
done; done
