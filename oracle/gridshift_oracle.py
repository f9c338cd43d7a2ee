"""CPU oracle for the MeanShift++ grid shift -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/gridshift/{grid,modeseek,track,segment}.py`).
It exists to *check* the CUDA engine and to time the reference CPU path in
`bench.py --impl reference` / the `cpu_baseline` leg.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` may import it; the product package
`paper_2104_00303_b200` never does, and has no CPU fallback.

Parity is pinned: `tests/golden/make_golden.py` runs the real reference
(importable in the build container) on seeded inputs and stores its
per-iteration cell tables, traces, labels and modes; `tests/test_oracle.py`
requires this restatement to reproduce every fixture bit for bit.

Every function cites the reference lines it follows.  The arithmetic uses the
same numpy primitives in the same order as the reference (IEEE divide then
floor, np.unique grouping, sequential np.bincount sums, offset-lexicographic
neighbour accumulation), so results are bitwise identical to it.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

# grid.py:22 -- lattice coordinates at or beyond this overflow the int64 keys
LATTICE_LIMIT = 2 ** 62
# modeseek.py:45 -- eta=None resolves to ETA_SCALE * n * h
ETA_SCALE = 1e-4
# track.py:26-27
WINDOW_TOL = 0.5
WINDOW_MAX_ITERS = 30


# ----------------------------------------------------------------- binning

def check_h(h) -> float:
    """grid.py:25-29: bandwidth must be finite and > 0."""
    h = float(h)
    if not (math.isfinite(h) and h > 0.0):
        raise ValueError(f"bandwidth must be a positive finite real, got {h!r}")
    return h


def bin_cells(y: np.ndarray, h: float) -> np.ndarray:
    """grid.py:78-85: int64 floor(y / h) with the 2^62 lattice guard."""
    h = check_h(h)
    q = np.floor(np.asarray(y, dtype=np.float64) / h)
    if q.size and float(np.abs(q).max()) >= LATTICE_LIMIT:
        raise ValueError("cell coordinates exceed the supported integer lattice; "
                         "bandwidth is too small for this coordinate range")
    return q.astype(np.int64)


def mixed_radix(cells: np.ndarray):
    """grid.py:137-158: padded row-major radix over this cell set.

    Returns (keys, strides) or None when prod(extents) >= 2^62.
    lo = per-axis min; every cell is shifted to start at 1 and the extent
    gets one spare slot on each side, so key(g+v) = key(g) + v.strides for
    v in {-1,0,1}^d.  Last axis varies fastest -> key order == lex order.
    """
    lo = cells.min(axis=0)
    shifted = cells - lo + 1
    extents = [int(e) for e in (shifted.max(axis=0) + 2)]
    prod = 1
    for e in extents:
        prod *= e
        if prod >= LATTICE_LIMIT:
            return None
    strides = np.ones(len(extents), dtype=np.int64)
    for j in range(len(extents) - 2, -1, -1):
        strides[j] = strides[j + 1] * extents[j + 1]
    return shifted @ strides, strides


def neighbour_offsets(d: int) -> np.ndarray:
    """grid.py:202-208: {-1,0,1}^d in itertools.product (lexicographic) order."""
    return np.array(list(itertools.product((-1, 0, 1), repeat=d)), dtype=np.int64)


# ------------------------------------------------------------------ tables

class Tables:
    """Occupied-cell tables, grid.py:88-134 (cells lexicographically sorted)."""

    def __init__(self, cells, counts, sums, keys, strides):
        self.cells = cells      # (k, d) int64
        self.counts = counts    # (k,) int64
        self.sums = sums        # (k, d) float64
        self.keys = keys        # (k,) int64 or None (overflow fallback)
        self.strides = strides  # (d,) int64 or None

    @property
    def k(self) -> int:
        return int(self.cells.shape[0])


def cell_tables(y: np.ndarray, h: float):
    """grid.py:161-190: group points by cell; counts and sequential fp64 sums.

    Returns (Tables, inverse) where inverse maps each point to its table row.
    """
    cells = bin_cells(y, h)
    radix = mixed_radix(cells)
    if radix is not None:
        pkeys, strides = radix
        ukeys, first, inverse, counts = np.unique(
            pkeys, return_index=True, return_inverse=True, return_counts=True)
        ucells = cells[first]
    else:  # grid.py:174-176 row-wise grouping
        ucells, inverse, counts = np.unique(
            cells, axis=0, return_inverse=True, return_counts=True)
        ukeys, strides = None, None
    inverse = inverse.reshape(-1)
    k, d = ucells.shape
    sums = np.empty((k, d), dtype=np.float64)
    for j in range(d):  # np.bincount adds in point order (grid.py:186-187)
        sums[:, j] = np.bincount(inverse, weights=y[:, j], minlength=k)
    return Tables(ucells, counts.astype(np.int64), sums, ukeys, strides), inverse


def neighbour_stats(t: Tables):
    """grid.py:230-273: 3^d-neighbourhood count and sum for every occupied cell.

    Neighbour contributions are accumulated in offset-lexicographic order,
    exactly as the chunked searchsorted + bincount of the reference does.
    """
    k, d = t.cells.shape
    out_c = np.zeros(k, dtype=np.int64)
    out_s = np.zeros((k, d), dtype=np.float64)
    if t.keys is not None:
        deltas = neighbour_offsets(d) @ t.strides
        m = deltas.size
        chunk = max(1, 4_000_000 // m)
        for a in range(0, k, chunk):
            b = min(a + chunk, k)
            q = (t.keys[a:b, None] + deltas[None, :]).ravel()
            pos = np.minimum(np.searchsorted(t.keys, q), k - 1)
            hit = t.keys[pos] == q
            rows = pos[hit]
            owner = np.nonzero(hit)[0] // m
            out_c[a:b] = np.bincount(owner, weights=t.counts[rows],
                                     minlength=b - a).astype(np.int64)
            for j in range(d):
                out_s[a:b, j] = np.bincount(owner, weights=t.sums[rows, j],
                                            minlength=b - a)
        return out_c, out_s
    where = {tuple(c): i for i, c in enumerate(t.cells.tolist())}
    offs = [tuple(v) for v in neighbour_offsets(d).tolist()]
    for i, c in enumerate(t.cells.tolist()):
        tot = 0
        acc = np.zeros(d)
        for v in offs:
            r = where.get(tuple(a + b for a, b in zip(c, v)))
            if r is not None:
                tot += int(t.counts[r])
                acc += t.sums[r]
        out_c[i] = tot
        out_s[i] = acc
    return out_c, out_s


def neighbour_aggregate(t: Tables, g):
    """grid.py:211-227: scalar 3^d aggregate around one query cell."""
    g = tuple(int(c) for c in g)
    if len(g) != t.cells.shape[1]:
        raise ValueError(f"query cell has dimension {len(g)}, tables have {t.cells.shape[1]}")
    where = {tuple(c): i for i, c in enumerate(t.cells.tolist())}
    tot = 0
    acc = np.zeros(len(g))
    for v in itertools.product((-1, 0, 1), repeat=len(g)):
        r = where.get(tuple(a + b for a, b in zip(g, v)))
        if r is not None:
            tot += int(t.counts[r])
            acc += t.sums[r]
    return tot, acc


# ------------------------------------------------------------------ engine

def shift_once(y: np.ndarray, h: float):
    """modeseek.py:105-111: y' = nbr_sums/nbr_counts per point; summed L2 move."""
    t, inverse = cell_tables(y, h)
    c, s = neighbour_stats(t)
    y_next = s[inverse] / c[inverse, None]
    movement = float(np.sqrt(((y_next - y) ** 2).sum(axis=1)).sum())
    return y_next, movement


def resolve_eta(eta, n: int, h: float) -> float:
    """modeseek.py:71-74."""
    return float(eta) if eta is not None else ETA_SCALE * n * h


def meanshiftpp(y: np.ndarray, h: float, eta=None, max_iters: int = 300,
                on_iter=None):
    """modeseek.py:125-146: loop until movement < eta (step applied) or cap.

    Returns dict(labels, k, modes, iterations, movement, converged, y).
    `on_iter(t, y_before)` is a test hook called before every shift.
    """
    h = check_h(h)
    y = np.ascontiguousarray(y, dtype=np.float64)
    thr = resolve_eta(eta, y.shape[0], h)
    hist = []
    converged = False
    for it in range(int(max_iters)):
        if on_iter is not None:
            on_iter(it, y)
        y, mv = shift_once(y, h)
        hist.append(mv)
        if mv < thr:
            converged = True
            break
    labels, k, modes = extract(y, h)
    return dict(labels=labels, k=k, modes=modes, iterations=len(hist),
                movement=np.asarray(hist, dtype=np.float64),
                converged=converged, y=y)


# -------------------------------------------------------------- extraction

def _find(parent, i):
    root = i
    while parent[root] != root:
        root = parent[root]
    while parent[i] != root:
        parent[i], i = root, parent[i]
    return root


def components(cells: np.ndarray) -> np.ndarray:
    """modeseek.py:204-253: union-find over Chebyshev-adjacent occupied cells.

    Returns the root row per cell (union by size, path compression; the root
    choice only matters through the first-appearance relabel downstream).
    """
    k, d = cells.shape
    parent = list(range(k))
    size = [1] * k

    def union(a, b):
        ra, rb = _find(parent, a), _find(parent, b)
        if ra == rb:
            return
        if size[ra] < size[rb]:
            ra, rb = rb, ra
        parent[rb] = ra
        size[ra] += size[rb]

    nonzero = [v for v in neighbour_offsets(d) if v.any()]
    radix = mixed_radix(cells)
    if radix is not None:
        keys, strides = radix
        for v in nonzero:
            delta = int(v @ strides)
            pos = np.minimum(np.searchsorted(keys, keys + delta), k - 1)
            for i in np.nonzero(keys[pos] == keys + delta)[0].tolist():
                union(i, int(pos[i]))
    else:
        where = {tuple(c): i for i, c in enumerate(cells.tolist())}
        for i, c in enumerate(cells.tolist()):
            for v in nonzero:
                j = where.get(tuple(a + b for a, b in zip(c, v.tolist())))
                if j is not None:
                    union(i, j)
    return np.asarray([_find(parent, i) for i in range(k)], dtype=np.int64)


def extract(y: np.ndarray, h: float):
    """modeseek.py:256-272: labels by first appearance, modes = label means."""
    cells = bin_cells(y, h)
    radix = mixed_radix(cells)
    if radix is not None:
        ukeys, first, inverse = np.unique(radix[0], return_index=True,
                                          return_inverse=True)
        ucells = cells[first]
    else:
        ucells, inverse = np.unique(cells, axis=0, return_inverse=True)
    comp = components(ucells)[inverse.reshape(-1)]
    ucomp, first_idx = np.unique(comp, return_index=True)
    rank = np.empty(ucomp.size, dtype=np.int64)
    rank[np.argsort(first_idx, kind="stable")] = np.arange(ucomp.size)
    labels = rank[np.searchsorted(ucomp, comp)]
    k = int(ucomp.size)
    cnt = np.bincount(labels, minlength=k).astype(np.float64)
    modes = np.empty((k, y.shape[1]))
    for j in range(y.shape[1]):
        modes[:, j] = np.bincount(labels, weights=y[:, j], minlength=k) / cnt
    return labels, k, modes


# ------------------------------------------------------------ segmentation

def image_to_features(pixels: np.ndarray, mode: str = "rgb", scale=None):
    """segment.py:77-92: uint8 (H,W,3) -> (H*W, 3|5) float64 rows."""
    pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
    hgt, wid = pixels.shape[:2]
    rgb = pixels.reshape(-1, 3).astype(np.float64)
    if mode == "rgb":
        return rgb
    if mode != "rgbxy":
        raise ValueError(f"mode must be one of ('rgb', 'rgbxy'), got {mode!r}")
    s = 255.0 / max(wid, hgt) if scale is None else float(scale)
    ys, xs = np.divmod(np.arange(hgt * wid), wid)
    return np.column_stack([rgb, xs * s, ys * s])


# ---------------------------------------------------------------- tracking

def window_rect(cx, cy, w, hp, fw, fh):
    """track.py:43-49: integer window rectangle clipped into the frame."""
    x0 = int(math.floor(cx - w / 2.0 + 0.5))
    y0 = int(math.floor(cy - hp / 2.0 + 0.5))
    x0 = min(max(x0, 0), max(fw - w, 0))
    y0 = min(max(y0, 0), max(fh - hp, 0))
    return x0, y0, min(x0 + w, fw), min(y0 + hp, fh)


def clamp_center(cx, cy, w, hp, fw, fh):
    """track.py:74-77."""
    return (min(max(cx, w / 2.0), fw - w / 2.0),
            min(max(cy, hp / 2.0), fh - hp / 2.0))


def colour_codes(bins: np.ndarray) -> np.ndarray:
    """track.py:92-94: (b0*2^20 + b1)*2^20 + b2."""
    return (bins[:, 0] * 2 ** 20 + bins[:, 1]) * 2 ** 20 + bins[:, 2]


def window_pixels(frame, rect):
    """track.py:80-85: window colours (f64) and absolute pixel coordinates."""
    x0, y0, x1, y1 = rect
    patch = frame[y0:y1, x0:x1].reshape(-1, 3).astype(np.float64)
    ys, xs = np.divmod(np.arange(patch.shape[0]), x1 - x0)
    return patch, xs + x0, ys + y0


def neighbourhood(bins: set) -> set:
    """track.py:138-144: N(B) = B + {-1,0,1}^3."""
    out = set()
    for b in bins:
        for v in neighbour_offsets(len(b)).tolist():
            out.add(tuple(a + o for a, o in zip(b, v)))
    return out


def track_frame(state: dict, frame: np.ndarray, h: float, update_bins=False,
                tol=WINDOW_TOL, max_iters=WINDOW_MAX_ITERS) -> dict:
    """track.py:147-188: re-centre on the mean (x, y) of bin-matching pixels.

    state = dict(cx, cy, w, hp, bins:set[tuple], lost, matches).
    """
    fh, fw = frame.shape[:2]
    cx, cy, w, hp = state["cx"], state["cy"], state["w"], state["hp"]
    codes_b = colour_codes(np.asarray(sorted(state["bins"]), dtype=np.int64))
    matches = 0
    for _ in range(max_iters):
        colours, xs, ys = window_pixels(frame, window_rect(cx, cy, w, hp, fw, fh))
        hit = np.isin(colour_codes(bin_cells(colours, h)), codes_b)
        matches = int(hit.sum())
        if matches == 0:
            return dict(state, lost=True, matches=0)
        nx, ny = float(xs[hit].mean()), float(ys[hit].mean())
        nx, ny = clamp_center(nx, ny, w, hp, fw, fh)
        moved = math.hypot(nx - cx, ny - cy)
        cx, cy = nx, ny
        if moved < tol:
            break
    bins = state["bins"]
    if update_bins:
        colours, _, _ = window_pixels(frame, window_rect(cx, cy, w, hp, fw, fh))
        seen = set(map(tuple, bin_cells(colours, h).tolist()))
        fresh = seen & neighbourhood(state["bins"])
        if fresh:
            bins = fresh
    return dict(state, cx=cx, cy=cy, bins=bins, lost=False, matches=matches)


def init_bins(frame: np.ndarray, cx, cy, w, hp, h, selected, eta=None,
              max_iters=300):
    """track.py:102-135: cluster the window colours, collect member cells."""
    fh, fw = frame.shape[:2]
    x0 = math.floor(cx - w / 2.0 + 0.5)
    y0 = math.floor(cy - hp / 2.0 + 0.5)
    if x0 < 0 or y0 < 0 or x0 + w > fw or y0 + hp > fh:
        raise ValueError("initial window must lie fully inside the frame")
    sel = sorted({int(c) for c in selected})
    if not sel:
        raise ValueError("select at least one cluster id")
    colours, _, _ = window_pixels(frame, window_rect(cx, cy, w, hp, fw, fh))
    res = meanshiftpp(colours, h, eta, max_iters)
    bad = [c for c in sel if c < 0 or c >= res["k"]]
    if bad:
        raise ValueError(f"cluster ids {bad} out of range, window has {res['k']} clusters")
    member = np.isin(res["labels"], sel)
    bins = set(map(tuple, bin_cells(colours[member], h).tolist()))
    return dict(cx=float(cx), cy=float(cy), w=int(w), hp=int(hp), bins=bins,
                lost=False, matches=int(member.sum()))


def track_sequence(frames, cx, cy, w, hp, h, selected, update_bins=False,
                   eta=None, max_iters=300):
    """track.py:191-205: one state row per frame; frozen after loss."""
    st = init_bins(frames[0], cx, cy, w, hp, h, selected, eta, max_iters)
    rows = [st]
    for fr in frames[1:]:
        if not st["lost"]:
            st = track_frame(st, fr, h, update_bins=update_bins)
        rows.append(st)
    return rows
