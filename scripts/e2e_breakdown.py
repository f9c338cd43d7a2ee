"""Where the end-to-end time goes (cfg4, 100M fp32 points): pinned H2D of the
input, the engine on device-resident input, pinned D2H of the labels, and the
host-API call that does all three (gs_meanshiftpp_host)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
x = W.cloud3d(n, seed=4)
cfg = gs.ShiftConfig(1.0, 1e-3, 50)
pts = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
pts.numpy()[:] = x
lab = torch.empty(n, dtype=torch.int64, pin_memory=True)
xd = torch.empty((n, 3), dtype=torch.float32, device="cuda")
ld = torch.empty(n, dtype=torch.int64, device="cuda")


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


h2d = t(lambda: xd.copy_(pts, non_blocking=True))
d2h = t(lambda: lab.copy_(ld, non_blocking=True))
dev = t(lambda: gs.meanshiftpp_device(xd, cfg, ld))
api = t(lambda: gs.meanshiftpp_points(pts.numpy(), cfg, labels_out=lab.numpy()))
print({"h2d_ms": h2d, "h2d_GBps": pts.numel() * 4 / h2d / 1e6, "d2h_ms": d2h,
       "d2h_GBps": lab.numel() * 8 / d2h / 1e6, "device_engine_ms": dev, "host_api_ms": api,
       "unexplained_ms": api - h2d - d2h - dev})
