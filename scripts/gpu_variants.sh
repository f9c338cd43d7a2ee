#!/bin/bash
# Time the engine with each variants/lib_*.so (GRIDSHIFT_LIB), plus a parity subset.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out
for lib in paper_2104_00303_b200/libgridshift_cuda.so variants/lib_*.so; do
  name=$(basename $lib .so)
  GRIDSHIFT_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/v_$name.json 2> $O/v_$name.err
  GRIDSHIFT_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/v_${name}_pytest.log 2>&1
  echo "$name $(tail -1 $O/v_${name}_pytest.log)"
done
