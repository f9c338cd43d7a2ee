"""Batched segmentation driver (paper_2104_00303_b200/batch.py, cfg2-style:
image i on rank i % world, no data-path collective) at world size 2 on CPU
(gloo) with an oracle-backed engine: every rank ends with the results of the
whole batch, in image order, equal to segmenting each image serially."""

import os
import socket
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_00303_b200 import workloads as W
from paper_2104_00303_b200.batch import local_indices, segment_batch
from paper_2104_00303_b200.modeseek import ShiftConfig, ShiftTrace
from paper_2104_00303_b200.segment import Image, SegmentMap

H, MODE, SCALE = 10.0, "rgbxy", 0.25


def _images():
    return [Image(W.voronoi_image(40, 24, 6, seed=70 + i)) for i in range(5)]


def oracle_engine(img, cfg, mode, scale):
    """segment_image restated on the oracle (segment.py:95-117)."""
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle import gridshift_oracle as O

    y = O.image_to_features(img.pixels, mode, scale)
    r = O.meanshiftpp(y, cfg.h, cfg.eta, cfg.max_iters)
    labels = r["labels"]
    rgb = img.pixels.reshape(-1, 3).astype(np.float64)
    cnt = np.bincount(labels, minlength=r["k"]).astype(np.float64)
    mean = np.column_stack([np.bincount(labels, weights=rgb[:, c], minlength=r["k"]) / cnt for c in range(3)])
    seg = SegmentMap(labels=labels.reshape(img.height, img.width), k=r["k"], mean_colors=mean)
    return seg, ShiftTrace(iterations=r["iterations"], total_movement_per_iter=np.asarray(r["movement"]),
                           converged=r["converged"])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []

    def engine(img, cfg, mode, scale):
        calls.append(img.pixels.tobytes())
        return oracle_engine(img, cfg, mode, scale)

    imgs = _images()
    res = segment_batch(imgs, ShiftConfig(h=H, eta=1e-3, max_iters=40), MODE, SCALE, engine=engine)
    mine = segment_batch(imgs, ShiftConfig(h=H, eta=1e-3, max_iters=40), MODE, SCALE, engine=oracle_engine,
                         gather=False)
    np.savez(Path(out) / f"r{rank}.npz", n_calls=len(calls), local=np.array(sorted(mine)),
             **{f"labels{i}": s.labels for i, (s, _) in enumerate(res)},
             **{f"k{i}": s.k for i, (s, _) in enumerate(res)},
             **{f"iters{i}": t.iterations for i, (_, t) in enumerate(res)})
    dist.destroy_process_group()


def test_batch_world2_equals_serial():
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        parts = [dict(np.load(Path(out) / f"r{r}.npz")) for r in range(2)]
    imgs = _images()
    ref = [oracle_engine(img, ShiftConfig(h=H, eta=1e-3, max_iters=40), MODE, SCALE) for img in imgs]
    for r, p in enumerate(parts):
        # each rank segmented only its own images (no duplicated work)
        assert int(p["n_calls"]) == len(local_indices(len(imgs), 2, r))
        assert p["local"].tolist() == local_indices(len(imgs), 2, r)
        for i, (seg, tr) in enumerate(ref):
            assert np.array_equal(p[f"labels{i}"], seg.labels)
            assert int(p[f"k{i}"]) == seg.k and int(p[f"iters{i}"]) == tr.iterations


def test_batch_single_process_and_ownership():
    imgs = _images()[:3]
    cfg = ShiftConfig(h=H, eta=1e-3, max_iters=40)
    res = segment_batch(imgs, cfg, MODE, SCALE, engine=oracle_engine)
    for img, (seg, _) in zip(imgs, res):
        want, _ = oracle_engine(img, cfg, MODE, SCALE)
        assert np.array_equal(seg.labels, want.labels)
    for count in (0, 1, 5, 8, 13):
        for world in (1, 2, 3, 8):
            owned = sorted(i for r in range(world) for i in local_indices(count, world, r))
            assert owned == list(range(count))


@pytest.mark.gpu
def test_batch_cuda_equals_segment_image():
    from paper_2104_00303_b200.segment import segment_image

    imgs = _images()[:3]
    cfg = ShiftConfig(h=H, eta=1e-3, max_iters=40)
    res = segment_batch(imgs, cfg, MODE, SCALE)
    for img, (seg, tr) in zip(imgs, res):
        want, wtr = segment_image(img, cfg, MODE, scale=SCALE)
        assert np.array_equal(seg.labels, want.labels) and tr.iterations == wtr.iterations
        ref, _ = oracle_engine(img, cfg, MODE, SCALE)
        assert np.array_equal(seg.labels, ref.labels)
