"""Row-sharded driver (paper_2104_00303_b200/sharded.py) at world sizes 2 and
4 on CPU (gloo), with the numpy shard backend: the sharded result must equal the
single-process exact-arithmetic model bit for bit (labels in global
first-appearance numbering, modes, movement trace, per-iteration tables)."""

import os
import socket
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_00303_b200 import workloads as W
from paper_2104_00303_b200.modeseek import ShiftConfig
from paper_2104_00303_b200.sharded import ShardLabels, meanshiftpp_sharded, shard_bounds
from tests import exact_model as X


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, y, h, eta, max_iters, out):
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from tests.shard_model import NumpyShard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(len(y), world, rank)
    be = NumpyShard(y[lo:hi])
    local, tr = meanshiftpp_sharded(torch.from_numpy(y[lo:hi]), ShiftConfig(h, eta, max_iters),
                                    n_total=len(y), backend=be, return_result=True)
    np.savez(Path(out) / f"r{rank}.npz", labels=local.labels, k=local.k, modes=local.modes,
             movement=tr.total_movement_per_iter, iters=tr.iterations, fp=tr.fingerprint_per_iter,
             offset=local.offset)
    dist.destroy_process_group()


CASES = {
    "blobs2d": (lambda: W.blobs2d(3001, seed=5), 0.5, 1e-4, 300),
    "cloud3d": (lambda: W.cloud3d(20_000, seed=6).astype(np.float64), 1.0, 1e-3, 12),
    "d4": (lambda: np.random.default_rng(3).normal(0, 1, size=(1500, 4)), 0.8, None, 300),
}


@pytest.mark.parametrize("name,world", [(n, 2) for n in sorted(CASES)] + [("cloud3d", 4)])
def test_sharded_equals_exact_model(name, world):
    gen, h, eta, mi = CASES[name]
    y = gen()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(world, _free_port(), y, h, eta, mi, out), nprocs=world, join=True)
        parts = [dict(np.load(Path(out) / f"r{r}.npz")) for r in range(world)]
    ref = X.meanshiftpp(y, h, eta, mi)
    for p in parts:
        assert int(p["iters"]) == ref["iterations"]
        np.testing.assert_array_equal(p["movement"], ref["movement"])
        assert [int(v) for v in p["fp"]] == [int(v) for v in ref["iter_fp"]]
        assert int(p["k"]) == ref["k"]
        assert np.array_equal(p["modes"], ref["modes"])
    labels = np.concatenate([p["labels"] for p in parts])
    assert np.array_equal(labels, ref["labels"])
    lab = ShardLabels(None, ref["k"], ref["modes"], 0).gather(
        [ShardLabels(p["labels"], int(p["k"]), p["modes"], int(p["offset"])) for p in parts])
    assert lab.k == ref["k"]


def test_shard_bounds_cover_rows():
    for n in (1, 7, 100, 12_345):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
