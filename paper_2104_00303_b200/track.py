"""Window tracking surface of the reference (`gridshift/track.py`).

`init_tracker` clusters the window colours with the CUDA MeanShift++ engine;
`track_sequence` / `track_frame` run the whole per-frame re-centring loop in
one persistent CTA (`gs_track_sequence`): colour-cell membership against a
bitmap of B, integer centroid reduction, clamp, tolerance test, and the
optional B <- cells(window) & N(B) refresh, all on device.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .grid import PointSet, bin_points
from .modeseek import Labeling, ShiftConfig, meanshiftpp
from .segment import Image

WINDOW_TOL = 0.5        # track.py:26
WINDOW_MAX_ITERS = 30   # track.py:27


@dataclass(frozen=True)
class Window:
    """track.py:30-49."""

    cx: float
    cy: float
    w: int
    h_px: int

    def __post_init__(self):
        if self.w < 1 or self.h_px < 1:
            raise ValueError(f"window extents must be positive, got {self.w}x{self.h_px}")

    def rect(self, frame_w: int, frame_h: int):
        x0 = int(math.floor(self.cx - self.w / 2.0 + 0.5))
        y0 = int(math.floor(self.cy - self.h_px / 2.0 + 0.5))
        x0 = min(max(x0, 0), max(frame_w - self.w, 0))
        y0 = min(max(y0, 0), max(frame_h - self.h_px, 0))
        return x0, y0, min(x0 + self.w, frame_w), min(y0 + self.h_px, frame_h)


@dataclass(frozen=True)
class BinSet:
    """track.py:52-61."""

    bins: frozenset
    h: float

    def __post_init__(self):
        if not self.bins:
            raise ValueError("bin set cannot be empty")


@dataclass(frozen=True)
class TrackState:
    """track.py:64-71."""

    window: Window
    bins: BinSet
    frame_w: int
    frame_h: int
    lost: bool = False
    last_match_count: int = 0


def _window_colors(frame: Image, win: Window) -> np.ndarray:
    x0, y0, x1, y1 = win.rect(frame.width, frame.height)
    return frame.pixels[y0:y1, x0:x1].reshape(-1, 3).astype(np.float64)


def cluster_window(frame: Image, window: Window, cfg: ShiftConfig) -> tuple[Labeling, np.ndarray]:
    """track.py:102-107 (engine on device)."""
    colors = _window_colors(frame, window)
    labeling, _ = meanshiftpp(PointSet(colors), cfg)
    return labeling, colors


def init_tracker(frame0: Image, window0: Window, cfg: ShiftConfig, selected_clusters) -> TrackState:
    """track.py:110-135."""
    x0 = math.floor(window0.cx - window0.w / 2.0 + 0.5)
    y0 = math.floor(window0.cy - window0.h_px / 2.0 + 0.5)
    if x0 < 0 or y0 < 0 or x0 + window0.w > frame0.width or y0 + window0.h_px > frame0.height:
        raise ValueError("initial window must lie fully inside the frame")
    selected = sorted({int(c) for c in selected_clusters})
    if not selected:
        raise ValueError("select at least one cluster id")
    labeling, colors = cluster_window(frame0, window0, cfg)
    bad = [c for c in selected if c < 0 or c >= labeling.k]
    if bad:
        raise ValueError(f"cluster ids {bad} out of range, window has {labeling.k} clusters")
    member = np.isin(labeling.labels, selected)
    cells = bin_points(colors[member], cfg.h)
    return TrackState(window=window0, bins=BinSet(bins=frozenset(map(tuple, cells.tolist())), h=cfg.h),
                      frame_w=frame0.width, frame_h=frame0.height, lost=False,
                      last_match_count=int(member.sum()))


def neighborhood(binset: BinSet) -> frozenset:
    """track.py:138-144: B dilated by {-1,0,1}^3."""
    out = set()
    for b in binset.bins:
        for v in np.ndindex(*(3,) * len(b)):
            out.add(tuple(a + o - 1 for a, o in zip(b, v)))
    return frozenset(out)


def _lattice(h: float) -> int:
    return int(math.floor(255.0 / h)) + 1


def _decode(bitmap_row: np.ndarray, L: int) -> frozenset:
    bits = np.unpackbits(bitmap_row.view(np.uint8), bitorder="little")[: L ** 3]
    codes = np.nonzero(bits)[0]
    a, rem = np.divmod(codes, L * L)
    b, c = np.divmod(rem, L)
    return frozenset(zip(a.tolist(), b.tolist(), c.tolist()))


def run_tracker(frames: np.ndarray, state: TrackState, h: float, update_bins: bool,
                tol: float = WINDOW_TOL, max_iters: int = WINDOW_MAX_ITERS, with_bins: bool = True):
    """Device loop over frames[1:] starting from `state` (frames[0] is the
    frame `state` belongs to).  Returns per-row arrays and per-row bin sets."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    T, H, W, _ = frames.shape
    if (W, H) != (state.frame_w, state.frame_h):
        raise ValueError(f"frame size {W}x{H} does not match the tracked sequence "
                         f"({state.frame_w}x{state.frame_h})")
    bins = np.asarray(sorted(state.bins.bins), dtype=np.int64).reshape(-1, 3)
    L = _lattice(h)
    words = (L ** 3 + 31) // 32
    cx = np.empty(T)
    cy = np.empty(T)
    lost = np.empty(T, dtype=np.int32)
    matches = np.empty(T, dtype=np.int64)
    nbins = np.empty(T, dtype=np.int64)
    hist = np.empty((T, words), dtype=np.uint32) if with_bins else None
    _lib.check(_lib.load().gs_track_sequence(
        _lib.context(), _lib.ptr(frames), T, H, W, float(state.window.cx), float(state.window.cy),
        int(state.window.w), int(state.window.h_px), _lib.ptr(bins), bins.shape[0], float(h),
        1 if update_bins else 0, int(state.last_match_count), float(tol), int(max_iters),
        _lib.ptr(cx), _lib.ptr(cy), _lib.ptr(lost), _lib.ptr(matches), _lib.ptr(nbins),
        _lib.ptr(hist)))
    rows_bins = [_decode(hist[t], L) for t in range(T)] if with_bins else None
    return cx, cy, lost.astype(bool), matches, nbins, rows_bins


def track_frame(state: TrackState, frame: Image, cfg: ShiftConfig, update_bins: bool = False,
                tol: float = WINDOW_TOL, max_iters: int = WINDOW_MAX_ITERS) -> TrackState:
    """track.py:147-188 for one frame (same device loop, one step)."""
    if state.lost:
        raise ValueError("tracker already lost the object")
    if (frame.width, frame.height) != (state.frame_w, state.frame_h):
        raise ValueError(f"frame size {frame.width}x{frame.height} does not match the "
                         f"tracked sequence ({state.frame_w}x{state.frame_h})")
    pair = np.stack([frame.pixels, frame.pixels])
    cx, cy, lost, matches, _, rows = run_tracker(pair, state, cfg.h, update_bins, tol, max_iters)
    if lost[1]:
        return replace(state, lost=True, last_match_count=0)
    return replace(state, window=replace(state.window, cx=float(cx[1]), cy=float(cy[1])),
                   bins=BinSet(bins=rows[1], h=state.bins.h), lost=False,
                   last_match_count=int(matches[1]))


def track_sequence(frames, window0: Window, cfg: ShiftConfig, selected_clusters,
                   update_bins: bool = False):
    """track.py:191-205: one TrackState per frame, frozen after loss."""
    imgs = [f if isinstance(f, Image) else Image(f) for f in frames]
    state = init_tracker(imgs[0], window0, cfg, selected_clusters)
    stack = np.stack([im.pixels for im in imgs])
    cx, cy, lost, matches, _, rows = run_tracker(stack, state, cfg.h, update_bins)
    out = [state]
    for t in range(1, len(imgs)):
        if lost[t]:
            prev = out[-1]
            out.append(replace(prev, lost=True, last_match_count=0))
        else:
            out.append(replace(state, window=replace(window0, cx=float(cx[t]), cy=float(cy[t])),
                               bins=BinSet(bins=rows[t], h=cfg.h), lost=False,
                               last_match_count=int(matches[t])))
    return out
