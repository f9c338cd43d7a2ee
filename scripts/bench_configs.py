"""Per-configuration device timings (not the driver's bench line): cfg0-cfg4
through the public device / host APIs, with the CUDA engine's per-kernel
accounting.  Usage: python scripts/bench_configs.py [cfg0 cfg1 cfg2 cfg3 cfg4]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import _lib
from paper_2104_00303_b200 import workloads as W


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    _lib.profile(1)
    t0 = time.perf_counter()
    out = None
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    prof = _lib.profile(2)
    _lib.profile(0)
    return out, dt, {k: round(v[0] / reps, 3) for k, v in prof.items() if v[1]}


def run_points(name, x, cfg):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    lab = torch.empty(len(x), dtype=torch.int64, device="cuda")
    (_, k, it, mv, conv), dt, prof = timed(lambda: gs.meanshiftpp_device(xd, cfg, lab))
    return {"config": name, "n": len(x), "d": x.shape[1], "iterations": it, "k": k,
            "ms": dt * 1e3, "point_updates_per_s": len(x) * it / dt, "kernels_ms": prof}


def main(which):
    res = []
    if "cfg0" in which:
        c = W.CONFIGS["cfg0"]
        res.append(run_points("cfg0", W.blobs2d(), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"])))
    if "cfg1" in which:
        c = W.CONFIGS["cfg1"]
        x = gs.image_to_features(gs.Image(W.cfg1_image()), "rgb").data
        res.append(run_points("cfg1", x, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"])))
    if "cfg2" in which:
        c = W.CONFIGS["cfg2"]
        x = gs.image_to_features(gs.Image(W.cfg2_image(0)), "rgbxy", 0.25).data
        res.append(run_points("cfg2 (one 4K image)", x, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"])))
    if "cfg3" in which:
        frames, cen, _ = W.tracking_video()
        win = gs.Window(cx=float(round(cen[0, 0])), cy=float(round(cen[0, 1])), w=128, h_px=128)
        cfg = gs.ShiftConfig(h=16.0)
        lab, colors = gs.cluster_window(gs.Image(frames[0]), win, cfg)
        x0, y0, x1, _ = win.rect(frames.shape[2], frames.shape[1])
        sel = int(lab.labels[(int(win.cy) - y0) * (x1 - x0) + int(win.cx) - x0])
        st = gs.init_tracker(gs.Image(frames[0]), win, cfg, [sel])
        from paper_2104_00303_b200.track import run_tracker
        out, dt, prof = timed(lambda: run_tracker(frames, st, 16.0, True, with_bins=False))
        cx, cy, lost, matches, nb, _ = out
        err = np.hypot(cx - cen[:, 0], cy - cen[:, 1])
        res.append({"config": "cfg3 tracking", "frames": len(frames), "ms": dt * 1e3,
                    "frames_per_s": len(frames) / dt, "lost_frames": int(lost.sum()),
                    "max_center_err_px": float(err.max()), "kernels_ms": prof})
    if "cfg4" in which:
        c = W.CONFIGS["cfg4"]
        res.append(run_points("cfg4", W.cloud3d(), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"])))
    for r in res:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
