"""Freeze the exact-arithmetic model (tests/exact_model.py) outputs for the
big configurations into big_<cfg>.npz (model_modes, model_movement,
model_labels_digest), next to the reference's own outputs.

    python tests/golden/make_model_golden.py cfg0 cfg1 cfg2 cfg4_10m
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from tests import exact_model as X  # noqa: E402
from tests.golden.exact_modes import inputs  # noqa: E402


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def main(name, cached=None):
    y, c = inputs(name)
    t0 = time.time()
    if cached and Path(cached).exists():
        r = dict(np.load(cached))
    else:
        r = X.meanshiftpp(y, c["h"], c["eta"], c["max_iters"])
    f = dict(np.load(HERE / f"big_{name}.npz"))
    f["model_modes"] = r["modes"]
    f["model_movement"] = np.asarray(r["movement"])
    f["model_labels_digest"] = np.asarray(digest(np.asarray(r["labels"], dtype=np.int64)))
    np.savez_compressed(HERE / f"big_{name}.npz", **f)
    print(json.dumps({"case": name, "model_vs_ref_modes_over_h":
                      float(np.abs(r["modes"] - f["modes"]).max() / c["h"]),
                      "labels_equal_ref": digest(np.asarray(r["labels"], dtype=np.int64)) == str(f["labels_digest"]),
                      "wall_s": time.time() - t0}))


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        main(nm, f"/tmp/model_{nm}.npz")
