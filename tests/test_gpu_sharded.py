"""CUDA shard backend (gs_shard_* C ABI) through the sharded driver.

World size 2 runs both ranks on cuda:0 with gloo collectives (host-staged;
no kernel waits on another rank's kernel), world size 1 uses NCCL.  Both
must equal the single-GPU engine bit for bit."""

import os
import socket
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2104_00303_b200 as gs
from paper_2104_00303_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, backend, y, h, eta, mi, out, order):
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2104_00303_b200.modeseek import ShiftConfig, set_sum_order
    from paper_2104_00303_b200.sharded import meanshiftpp_sharded, shard_bounds

    set_sum_order(order)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    lo, hi = shard_bounds(len(y), world, rank)
    x = torch.from_numpy(y[lo:hi]).cuda()
    local, tr = meanshiftpp_sharded(x, ShiftConfig(h, eta, mi), n_total=len(y), return_result=True)
    np.savez(Path(out) / f"r{rank}.npz", labels=local.labels, k=local.k, modes=local.modes,
             movement=tr.total_movement_per_iter, iters=tr.iterations, fp=tr.fingerprint_per_iter)
    dist.destroy_process_group()


@pytest.mark.parametrize("order", ["seqmodel", "exact"])
@pytest.mark.parametrize("world,backend,n", [(1, "nccl", 200_000), (2, "gloo", 200_000), (2, "gloo", 5_000)])
def test_cuda_shards_equal_single_gpu(world, backend, n, order):
    """Sharded runs equal the single-GPU engine bit for bit in the default
    sum order (the sequential model is a function of the merged cell table
    only, so every rank computes the same sums) and in the exact order."""
    y = W.cloud3d(n, seed=21)
    h, eta, mi = 1.0, 1e-3, 20
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(world, _free_port(), backend, y, h, eta, mi, out, order), nprocs=world, join=True)
        parts = [dict(np.load(Path(out) / f"r{r}.npz")) for r in range(world)]
    with gs.sum_order(order):
        lab, tr = gs.meanshiftpp(gs.PointSet(y.astype(np.float64)), gs.ShiftConfig(h, eta, mi))
    for p in parts:
        assert int(p["iters"]) == tr.iterations
        np.testing.assert_array_equal(p["movement"], tr.total_movement_per_iter)
        assert [int(v) for v in p["fp"]] == [int(v) for v in tr.fingerprint_per_iter]
        assert np.array_equal(p["modes"], lab.modes)
    assert np.array_equal(np.concatenate([p["labels"] for p in parts]), lab.labels)
