import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import workloads as W, _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
x = W.cloud3d(n)
cfg = gs.ShiftConfig(h=1.0, eta=1e-3, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 50)
xd = torch.from_numpy(x).cuda()
lab, k, it, mv, conv = gs.meanshiftpp_device(xd, cfg)
torch.cuda.synchronize()
l = lab.cpu().numpy()
print("device api: k", k, "iters", it, "min", l.min(), "max", l.max(), "nuniq", len(np.unique(l)), flush=True)
pts = x.astype(np.float64)
out = np.empty(n, dtype=np.int64)
try:
    L2, tr = gs.meanshiftpp(gs.PointSet(pts), cfg, labels_out=out)
    print("host api ok: k", L2.k, "iters", tr.iterations, flush=True)
except ValueError as e:
    print("host api error", e, "min", out.min(), "max", out.max(), "nuniq", len(np.unique(out)), flush=True)
print("equal labels:", np.array_equal(out, l), flush=True)
