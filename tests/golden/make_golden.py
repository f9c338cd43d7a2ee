"""Generate golden fixtures by running the REAL reference (gridshift) here.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

The reference is pure Python/numpy and is importable
in the build container only; it does not exist on the GPU box, so its outputs
are frozen into `tests/golden/*.npz` and the GPU parity tests read those.

Small fixtures (always): cell tables + neighbour stats, single steps, full
engine runs with per-iteration table fingerprints, extraction, tracking.
Big fixtures (--big): cfg0 and cfg1 at full BASELINE size with labels and
modes; cfg2 (one 4K image) and cfg4 at 10M points with labels/modes digests.
"""

from __future__ import annotations

import argparse
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import gridshift.modeseek as ms  # noqa: E402
from gridshift import grid, track  # noqa: E402
from gridshift.grid import PointSet  # noqa: E402
from gridshift.modeseek import ShiftConfig, extract_clusters, meanshiftpp, meanshiftpp_step  # noqa: E402
from gridshift.segment import Image, image_to_features  # noqa: E402
from gridshift.synthetic import drift_frames, moving_square_frames, removal_frames  # noqa: E402

from paper_2104_00303_b200 import workloads as W  # noqa: E402


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


class Recorder:
    """Wraps grid._tables_from_data as seen by modeseek to log every
    iteration's (k, fingerprint(cells, counts))."""

    def __init__(self):
        self.ks, self.fps = [], []
        self._orig = ms._tables_from_data

    def __enter__(self):
        def wrapped(data, h):
            t, inv = self._orig(data, h)
            self.ks.append(t.cells.shape[0])
            self.fps.append(W.fingerprint(t.cells, t.counts))
            return t, inv
        ms._tables_from_data = wrapped
        return self

    def __exit__(self, *exc):
        ms._tables_from_data = self._orig


def run_engine(y, h, eta, max_iters):
    with Recorder() as rec:
        lab, tr = meanshiftpp(PointSet(y), ShiftConfig(h=h, eta=eta, max_iters=max_iters))
    return dict(labels=lab.labels, k=np.int64(lab.k), modes=lab.modes,
                iterations=np.int64(tr.iterations), movement=tr.total_movement_per_iter,
                converged=np.bool_(tr.converged),
                iter_k=np.asarray(rec.ks, dtype=np.int64),
                iter_fp=np.asarray(rec.fps, dtype=np.uint64))


def put(store, case, **fields):
    for k, v in fields.items():
        store[f"{case}__{k}"] = np.asarray(v)


# ---------------------------------------------------------------- groups

def make_tables(store):
    rng = np.random.default_rng(2024)
    cases = [
        ("singleton", np.array([[0.3, 0.3]]), 1.0),
        ("three_two", np.array([[0.1], [0.9], [1.1]]), 1.0),
        ("negative", np.array([[-0.1, -0.1], [-0.9, -1.5]]), 1.0),
        ("uniform3d", rng.uniform(0, 1, size=(1000, 3)), 0.25),
        ("normal2d", rng.normal(0, 1, size=(300, 2)), 0.4),
        ("normal3d", rng.normal(0, 1, size=(500, 3)), 0.5),
        ("d1", rng.normal(0, 3, size=(700, 1)), 0.3),
        ("d4", rng.normal(0, 1, size=(600, 4)), 0.7),
        ("d5", rng.normal(0, 1, size=(800, 5)), 0.9),
        ("d6", rng.normal(0, 1, size=(400, 6)), 1.1),
    ]
    # points parked exactly on cell faces (test_acceptance.py:58-61 idiom)
    faces = rng.normal(0, 4, size=(400, 3))
    faces[:200] = np.round(faces[:200] / 0.5) * 0.5
    cases.append(("faces3d", faces, 0.5))
    clipped = np.clip(np.floor(rng.normal(128, 90, size=(900, 3)) + 0.5), 0, 255)
    cases.append(("clipped_rgb", clipped, 8.0))
    names = []
    for name, y, h in cases:
        t, inv = grid._tables_from_data(y, h)
        nc, ns = grid._neighbor_stats_cells(t)
        put(store, f"tables_{name}", y=y, h=h, cells=t.cells, counts=t.counts, sums=t.sums,
            inverse=inv, nbr_counts=nc, nbr_sums=ns)
        names.append(f"tables_{name}")
    store["tables__names"] = np.array(names)


def make_steps(store):
    """200-instance criterion-1 generator (test_acceptance.py:38-61), trimmed
    to n <= 600 so the fixture stays small."""
    rng = np.random.default_rng(11)
    names = []
    for trial in range(120):
        d = int(rng.integers(1, 6))
        n = int(rng.integers(1, 601))
        scale = float(10.0 ** rng.uniform(-1.0, 2.0))
        h = float(scale * 10.0 ** rng.uniform(-1.5, 0.5))
        y = rng.normal(0.0, scale, size=(n, d))
        if trial % 3 == 0:
            y[: n // 2] = np.round(y[: n // 2] / h) * h
        moved, mv = meanshiftpp_step(PointSet(y), ShiftConfig(h=h))
        put(store, f"step_{trial}", y=y, h=h, y_next=moved.data, movement=mv)
        names.append(f"step_{trial}")
    store["steps__names"] = np.array(names)


def two_blobs(n_per, sep=2.0, sigma=0.05, seed=0, d=2):
    rng = np.random.default_rng(seed)
    a = rng.normal(0.0, sigma, size=(n_per, d))
    b = rng.normal(0.0, sigma, size=(n_per, d))
    b[:, 0] += sep
    return np.vstack([a, b])


def make_runs(store):
    rng = np.random.default_rng(77)
    img_rgb = W.voronoi_image(160, 120, 12, seed=5)
    img_xy = W.voronoi_image(160, 120, 16, seed=6)
    cases = [
        ("two_blobs", two_blobs(100, seed=5), 0.3, None, 300),
        ("two_blobs_cap", two_blobs(50, seed=9), 0.3, 1e-300, 3),
        ("identical", np.tile([1.5, -0.5, 2.0], (40, 1)), 0.7, None, 300),
        ("fixed_point", np.array([[0.2], [9.7]]), 1.0, None, 300),
        ("huge_h", rng.uniform(0, 1, size=(120, 3)), 50.0, None, 300),
        ("blobs2d_5k", W.blobs2d(5000, seed=3), 0.5, 1e-4, 300),
        ("rgb_small", image_to_features(Image(img_rgb), "rgb").data, 8.0, 1e-3, 100),
        ("rgbxy_small", image_to_features(Image(img_xy), "rgbxy", scale=0.25).data, 10.0, 1e-3, 100),
        ("cloud_50k", W.cloud3d(50_000, seed=8).astype(np.float64), 1.0, 1e-3, 50),
        ("d4_mix", np.vstack([rng.normal(c, 0.3, size=(300, 4)) for c in (0.0, 3.0, 6.0)]), 0.6, None, 300),
        ("d5_auto_eta", rng.normal(0, 1, size=(2000, 5)), 0.8, None, 300),
        ("d1_line", rng.normal(0, 2, size=(3000, 1)), 0.25, None, 300),
    ]
    names = []
    for name, y, h, eta, mi in cases:
        r = run_engine(y, h, eta, mi)
        put(store, f"run_{name}", y=y, h=h, eta=(np.nan if eta is None else eta),
            max_iters=mi, **r)
        names.append(f"run_{name}")
    store["runs__names"] = np.array(names)


def make_extract(store):
    rng = np.random.default_rng(31)
    cases = [
        ("two_groups", np.array([[0.1], [0.2], [2.3], [2.4]]), 1.0),
        ("adjacent", np.array([[0.95], [1.05]]), 1.0),
        ("diagonal", np.array([[0.9, 0.9], [1.1, 1.1]]), 1.0),
        ("first_appearance", np.array([[5.5], [0.1], [5.6], [9.9]]), 1.0),
        ("chain", np.arange(6, dtype=float).reshape(-1, 1) + 0.5, 1.0),
        ("means", np.vstack([rng.normal(0, 0.02, (30, 2)), rng.normal(5, 0.02, (20, 2))]), 0.5),
        ("random2d", rng.uniform(-3, 3, size=(400, 2)), 0.5),
        ("random3d", rng.uniform(-3, 3, size=(3000, 3)), 0.4),
    ]
    names = []
    for name, y, h in cases:
        lab = extract_clusters(PointSet(y), h)
        put(store, f"extract_{name}", y=y, h=h, labels=lab.labels, k=lab.k, modes=lab.modes)
        names.append(f"extract_{name}")
    store["extract__names"] = np.array(names)


def _track_rows(rows):
    cx = np.array([r.window.cx for r in rows])
    cy = np.array([r.window.cy for r in rows])
    lost = np.array([r.lost for r in rows])
    matches = np.array([r.last_match_count for r in rows], dtype=np.int64)
    nb = np.array([len(r.bins.bins) for r in rows], dtype=np.int64)
    fp = np.array([W.fingerprint(np.array(sorted(r.bins.bins), dtype=np.int64),
                                 np.zeros(len(r.bins.bins), dtype=np.int64)) for r in rows],
                  dtype=np.uint64)
    return dict(cx=cx, cy=cy, lost=lost, matches=matches, nbins=nb, bins_fp=fp)


def _object_id(frame, win, cfg):
    lab, _ = track.cluster_window(frame, win, cfg)
    x0, y0, x1, _ = win.rect(frame.width, frame.height)
    return int(lab.labels[(int(win.cy) - y0) * (x1 - x0) + int(win.cx) - x0])


def make_tracking(store):
    cfg = ShiftConfig(h=32.0)
    names = []

    def add(name, frames, win, h, update):
        cfg_ = ShiftConfig(h=h)
        obj = _object_id(frames[0], win, cfg_)
        rows = track.track_sequence(frames, win, cfg_, [obj], update_bins=update)
        put(store, f"track_{name}", frames=np.stack([f.pixels for f in frames]),
            win=np.array([win.cx, win.cy, win.w, win.h_px]), h=h, update=update,
            selected=obj, **_track_rows(rows))
        names.append(f"track_{name}")

    fr, _ = moving_square_frames(n_frames=30, width=160)
    add("square", fr, track.Window(cx=22.0, cy=45.0, w=31, h_px=31), 32.0, False)
    fr, _ = removal_frames(n_present=4, n_absent=3)
    add("removal", fr, track.Window(cx=60.0, cy=45.0, w=31, h_px=31), 32.0, False)
    fr, _ = drift_frames(n_frames=20)
    add("drift_upd", fr, track.Window(cx=60.0, cy=45.0, w=25, h_px=25), 32.0, True)
    add("drift_frozen", fr, track.Window(cx=60.0, cy=45.0, w=25, h_px=25), 32.0, False)
    vid, cen, _ = W.tracking_video(n_frames=40, width=320, height=240, seed=9, axes=(30, 20))
    frames = [Image(v) for v in vid]
    add("video_small", frames, track.Window(cx=float(round(cen[0, 0])), cy=float(round(cen[0, 1])),
                                           w=64, h_px=64), 16.0, True)
    store["track__names"] = np.array(names)
    del cfg


def make_cfg3_full(out_dir: Path):
    """cfg3 at BASELINE size: 300 frames of 1280x720, 128x128 window on the
    object, h=16, B updated every frame (track.py:191-205).  Frames are not
    stored: the GPU test regenerates them from workloads.tracking_video."""
    vid, cen, _ = W.tracking_video()
    frames = [Image(v) for v in vid]
    win = track.Window(cx=float(round(cen[0, 0])), cy=float(round(cen[0, 1])), w=128, h_px=128)
    cfg = ShiftConfig(h=16.0)
    obj = _object_id(frames[0], win, cfg)
    t0 = time.time()
    rows = track.track_sequence(frames, win, cfg, [obj], update_bins=True)
    wall = time.time() - t0
    np.savez_compressed(out_dir / "big_cfg3_full.npz", win=np.array([win.cx, win.cy, win.w, win.h_px]),
                        h=16.0, selected=obj, wall_s=wall, frames_digest=digest(vid),
                        **_track_rows(rows))


def make_big(out_dir: Path, which):
    for name in which:
        t0 = time.time()
        if name == "cfg0":
            y = W.blobs2d()
            c = W.CONFIGS["cfg0"]
        elif name == "cfg1":
            y = image_to_features(Image(W.cfg1_image()), "rgb").data
            c = W.CONFIGS["cfg1"]
        elif name == "cfg2":
            y = image_to_features(Image(W.cfg2_image(0)), "rgbxy", scale=0.25).data
            c = W.CONFIGS["cfg2"]
        elif name.startswith("cfg2_img"):
            y = image_to_features(Image(W.cfg2_image(int(name[8:]))), "rgbxy", scale=0.25).data
            c = W.CONFIGS["cfg2"]
        elif name == "cfg4_10m":
            y = W.cloud3d(10_000_000).astype(np.float64)
            c = W.CONFIGS["cfg4"]
        elif name == "cfg4_100m":
            y = W.cloud3d(100_000_000).astype(np.float64)
            c = W.CONFIGS["cfg4"]
        elif name == "cfg3_full":
            make_cfg3_full(out_dir)
            print(f"cfg3_full {time.time() - t0:.1f}s", flush=True)
            continue
        else:
            raise SystemExit(f"unknown big case {name}")
        r = run_engine(y, c["h"], c["eta"], c["max_iters"])
        wall = time.time() - t0
        lab = r.pop("labels")
        small = lab.max() < 65536
        fields = dict(r, labels_digest=digest(lab), modes_digest=digest(r["modes"]),
                      n=y.shape[0], d=y.shape[1], wall_s=wall)
        if small and not name.startswith("cfg4"):
            fields["labels_u16"] = lab.astype(np.uint16)
        if name == "cfg4_100m":
            fields["label_sizes"] = np.bincount(lab, minlength=int(r["k"]))
        n_rows, d_cols = y.shape
        del y
        np.savez_compressed(out_dir / f"big_{name}.npz", **{k: np.asarray(v) for k, v in fields.items()})
        print(f"{name}: n={n_rows} iters={int(r['iterations'])} k={int(r['k'])} {wall:.1f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", nargs="*", default=None)
    ap.add_argument("--skip-small", action="store_true")
    a = ap.parse_args()
    if not a.skip_small:
        for group, fn in [("tables", make_tables), ("steps", make_steps), ("runs", make_runs),
                          ("extract", make_extract), ("tracking", make_tracking)]:
            store = {}
            t0 = time.time()
            fn(store)
            np.savez_compressed(HERE / f"{group}.npz", **store)
            print(f"{group}: {len(store)} arrays, {time.time() - t0:.1f}s", flush=True)
    if a.big is not None:
        make_big(HERE, a.big or ["cfg0", "cfg1"])


if __name__ == "__main__":
    main()
