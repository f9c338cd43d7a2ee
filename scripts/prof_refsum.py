"""Profile one cfg4-shaped run (n points, max_iters) for ncu launch lists:
python scripts/prof_refsum.py [n] [iters] [exact]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if len(sys.argv) > 3 and sys.argv[3] == "exact":
    gs.set_sum_order("exact")
x = torch.from_numpy(W.cloud3d(n)).cuda()
lab = torch.empty(n, dtype=torch.int64, device="cuda")
cfg = gs.ShiftConfig(1.0, 1e-3, iters)
gs.meanshiftpp_device(x, cfg, lab)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_, k, it, mv, conv = gs.meanshiftpp_device(x, cfg, lab)
e1.record()
torch.cuda.synchronize()
print(f"n={n} iters={it} k={k} ms={e0.elapsed_time(e1):.3f}")
if not (len(sys.argv) > 3 and sys.argv[3] == "exact"):
    st = gs.modeseek.last_refsum_stats(it)
    print("table  nseg  nbig  nelem  maxlen  recomputed")
    for t, row in enumerate(st):
        print(t, *row.tolist())
