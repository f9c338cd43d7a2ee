"""Small end-to-end exercise of every engine entry point, for
compute-sanitizer runs (memcheck / racecheck / synccheck, one tool per run)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import workloads as W

rng = np.random.default_rng(0)
# dense d=3 with the spatial sort (n >= 32768), collapsed and per-point
x = W.cloud3d(40_000, seed=3).astype(np.float64)
cfg = gs.ShiftConfig(1.0, 1e-3, 8)
lab, tr = gs.meanshiftpp(gs.PointSet(x), cfg)
xd = torch.from_numpy(x).cuda()
gs.meanshiftpp_device(xd, cfg, collapsed=True)
# hash tables, d=5, sorted
img = gs.Image(W.voronoi_image(256, 160, 12, seed=2))
gs.segment_pixels(img, gs.ShiftConfig(10.0, 1e-3, 10), "rgbxy", 0.25)
# small unsorted cases, d = 1..6
for d in range(1, 7):
    y = rng.normal(0, 1, size=(500, d))
    gs.meanshiftpp(gs.PointSet(y), gs.ShiftConfig(0.7))
    gs.meanshiftpp_step(gs.PointSet(y), gs.ShiftConfig(0.7))
    gs.neighbor_stats(gs.PointSet(y), 0.7)
    gs.extract_clusters(gs.PointSet(y), 0.7)
# tracker
f, cen, _ = W.tracking_video(n_frames=6, width=200, height=160, seed=4, axes=(20, 14))
win = gs.Window(cx=float(round(cen[0, 0])), cy=float(round(cen[0, 1])), w=48, h_px=48)
lb, _ = gs.cluster_window(gs.Image(f[0]), win, gs.ShiftConfig(16.0))
gs.track_sequence([gs.Image(p) for p in f], win, gs.ShiftConfig(16.0), [0], update_bins=True)
torch.cuda.synchronize()
print("sanitize smoke ok", lab.k, tr.iterations)
