"""Deviation of each sum order from the reference fixtures, per configuration:
python scripts/sum_modes_check.py [mode ...] -- for cfg0, cfg1, cfg2 (image 0),
cfg4@10M and cfg4@100M: per-iteration (cells, counts) fingerprints equal?,
labels equal?, max |modes - reference| / h, device ms per run."""
import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import workloads as W
from tests import goldens as G


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def one(name, x, cfg, f, h):
    t0 = time.perf_counter()
    lab, tr = gs.meanshiftpp_points(x, cfg)
    dt = time.perf_counter() - t0
    fp_ok = [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in f["iter_fp"]]
    if "labels_u16" in f:
        lab_ok = bool(np.array_equal(lab.labels, f["labels_u16"].astype(np.int64)))
    else:
        lab_ok = digest(lab.labels) == str(f["labels_digest"])
    dev = float(np.abs(lab.modes - f["modes"]).max()) / h if lab.modes.shape == f["modes"].shape else None
    return {"config": name, "iterations": tr.iterations, "ref_iterations": int(f["iterations"]),
            "fingerprints_equal": fp_ok, "labels_equal": lab_ok, "modes_dev_over_h": dev,
            "host_call_s": round(dt, 3)}


def main(modes, which):
    for mode in modes:
        with gs.sum_order(mode):
            for w in which:
                if w == "cfg0":
                    c = W.CONFIGS["cfg0"]
                    r = one(w, W.blobs2d(), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), G.big("cfg0"), c["h"])
                elif w == "cfg1":
                    c = W.CONFIGS["cfg1"]
                    x = gs.image_to_features(gs.Image(W.cfg1_image()), "rgb").data
                    r = one(w, x, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), G.big("cfg1"), c["h"])
                elif w == "cfg2":
                    c = W.CONFIGS["cfg2"]
                    x = gs.image_to_features(gs.Image(W.cfg2_image(0)), "rgbxy", 0.25).data
                    r = one(w, x, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), G.big("cfg2"), c["h"])
                elif w == "cfg4_10m":
                    c = W.CONFIGS["cfg4"]
                    x = W.cloud3d(10_000_000).astype(np.float64)
                    r = one(w, x, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), G.big("cfg4_10m"), c["h"])
                else:
                    c = W.CONFIGS["cfg4"]
                    r = one(w, W.cloud3d(), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), G.big("cfg4_100m"), c["h"])
                r["sum_order"] = mode
                print(json.dumps(r), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    modes = [a for a in args if a in gs.modeseek.SUM_ORDERS] or ["reference", "exact", "seqmodel"]
    which = [a for a in args if a.startswith("cfg")] or ["cfg0", "cfg1", "cfg2", "cfg4_10m", "cfg4_100m"]
    main(modes, which)
