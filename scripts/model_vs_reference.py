"""Sequential-model sums against reference-order sums on the GPU: the max
iterate difference after 1, 2, ... iterations
(python scripts/model_vs_reference.py n [f32|f64] [shuffled|sorted|blocks]).
`sorted`: rows sorted along x (the least well-mixed point order there is);
`blocks`: rows grouped by generating component (cluster by cluster)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
dt = sys.argv[2] if len(sys.argv) > 2 else "f32"
order = sys.argv[3] if len(sys.argv) > 3 else "shuffled"
x = W.cloud3d(n)
if dt == "f64":
    x = x.astype(np.float64)
if order == "sorted":
    x = np.ascontiguousarray(x[np.argsort(x[:, 0], kind="stable")])
elif order == "blocks":
    x = np.ascontiguousarray(x[np.lexsort((x[:, 2], np.floor(x[:, 1] / 7.0), np.floor(x[:, 0] / 7.0)))])
xd = torch.from_numpy(x).cuda()
lab = torch.empty(n, dtype=torch.int64, device="cuda")
for iters in (1, 2, 3, 4, 6, 10, 50):
    cfg = gs.ShiftConfig(1.0, 1e-3, iters)
    ys = {}
    for mode in ("reference", "seqmodel"):
        with gs.sum_order(mode):
            gs.meanshiftpp_device(xd, cfg, lab)
            ys[mode] = gs.modeseek.last_iterate(n, 3)
    d = np.abs(ys["reference"] - ys["seqmodel"])
    i = int(d.max(axis=1).argmax())
    print(f"n={n} {dt} {order} iters={iters}: max|dy|={d.max():.3e} rows differing={int((d.max(axis=1) > 0).sum())} "
          f"worst row {i}: ref={ys['reference'][i]} model={ys['seqmodel'][i]}", flush=True)
