"""How much do the reference's modes move when only the fp64 summation order
changes?  Runs the reference algorithm (oracle restatement, bitwise-pinned)
on cfg4 at 10M points in its original row order and in a shuffled row order,
maps clusters through the (identical) partitions and reports max |dmodes|/h.

    python tests/golden/order_sensitivity.py > tests/golden/order_sensitivity.json
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle import gridshift_oracle as O  # noqa: E402
from paper_2104_00303_b200 import workloads as W  # noqa: E402


def main(n=10_000_000, seed=99):
    c = W.CONFIGS["cfg4"]
    y = W.cloud3d(n).astype(np.float64)
    t0 = time.time()
    a = O.meanshiftpp(y, c["h"], c["eta"], c["max_iters"])
    perm = np.random.default_rng(seed).permutation(n)
    b = O.meanshiftpp(y[perm], c["h"], c["eta"], c["max_iters"])
    la = a["labels"]
    lb = np.empty_like(la)
    lb[perm] = b["labels"]
    # the partitions must agree; map b's clusters onto a's
    first = {}
    mapping = np.full(b["k"], -1, dtype=np.int64)
    mapping[lb] = la
    same_partition = bool(np.array_equal(mapping[lb], la)) and a["k"] == b["k"]
    dm = np.abs(a["modes"][mapping] - b["modes"]).max() / c["h"]
    out = {"n": n, "iterations": [a["iterations"], b["iterations"]], "k": [a["k"], b["k"]],
           "same_partition": same_partition, "max_dmodes_over_h": float(dm),
           "dmodes_quantiles_over_h": [float(q) for q in np.quantile(
               np.abs(a["modes"][mapping] - b["modes"]).max(axis=1) / c["h"], [0.5, 0.99, 0.999, 1.0])],
           "wall_s": time.time() - t0}
    del first
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(int(v) for v in sys.argv[1:]))
