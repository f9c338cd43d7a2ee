"""Augment big_<cfg>.npz with the exactly rounded modes of the REFERENCE's
own final iterate: modes_exact[c] = fsum(y_final[labels == c]) / count.

The reference computes modes with a sequential np.bincount
(modeseek.py:268-271); summing ~1e6 identical fp64 positions one by one
accumulates a systematic rounding bias that reordering cannot reveal.  This
script measures it, so the parity test can state both distances.

    python tests/golden/exact_modes.py cfg4_10m
"""
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from oracle import gridshift_oracle as O  # noqa: E402
from paper_2104_00303_b200 import workloads as W  # noqa: E402


def inputs(name):
    from paper_2104_00303_b200.segment import Image, image_to_features
    if name == "cfg0":
        return W.blobs2d(), W.CONFIGS["cfg0"]
    if name == "cfg1":
        return image_to_features(Image(W.cfg1_image()), "rgb").data, W.CONFIGS["cfg1"]
    if name == "cfg2":
        return image_to_features(Image(W.cfg2_image(0)), "rgbxy", 0.25).data, W.CONFIGS["cfg2"]
    if name == "cfg4_10m":
        return W.cloud3d(10_000_000).astype(np.float64), W.CONFIGS["cfg4"]
    raise SystemExit(name)


def main(name):
    y, c = inputs(name)
    r = O.meanshiftpp(y, c["h"], c["eta"], c["max_iters"])
    yf, lab, k = r["y"], r["labels"], r["k"]
    order = np.argsort(lab, kind="stable")
    bounds = np.searchsorted(lab[order], np.arange(k + 1))
    exact = np.empty((k, y.shape[1]))
    for ci in range(k):
        idx = order[bounds[ci]:bounds[ci + 1]]
        for j in range(y.shape[1]):
            exact[ci, j] = math.fsum(yf[idx, j]) / len(idx)
    f = dict(np.load(HERE / f"big_{name}.npz"))
    assert np.array_equal(f["modes"], r["modes"]), "oracle must reproduce the reference modes"
    f["modes_exact"] = exact
    np.savez_compressed(HERE / f"big_{name}.npz", **f)
    dev = np.abs(r["modes"] - exact).max() / c["h"]
    print(json.dumps({"case": name, "k": int(k), "max_ref_minus_exact_over_h": float(dev)}))


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        main(nm)
