"""Point sets, binning and cell tables -- the grid surface of the reference
(`gridshift/grid.py`), with the table builds running on the B200.

`build_cell_tables` and `neighbor_stats` go through `gs_build_tables`
(include/gridshift_cuda.h): one fused bin + key + exact-sum histogram kernel
and the 3^d neighbour aggregation kernel.  Counts are bit-exact against the
reference; sums are exact-then-rounded (the reference sums sequentially in
fp64, grid.py:186-187), which the reference's own tests accept at rtol 1e-9.
"""

from __future__ import annotations

import ctypes as C
import itertools
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

GridIndex = tuple

# grid.py:22
COORD_LIMIT = 2 ** 62


def check_bandwidth(h) -> float:
    """grid.py:25-29."""
    h = float(h)
    if not math.isfinite(h) or h <= 0.0:
        raise ValueError(f"bandwidth must be a positive finite real, got {h!r}")
    return h


@dataclass
class PointSet:
    """n points in d-dimensional feature space (grid.py:32-59): data is a
    C-contiguous float64 (n, d) array, n, d >= 1, all entries finite."""

    data: np.ndarray

    def __post_init__(self):
        arr = np.ascontiguousarray(self.data, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError(f"point data must be 2-d (n, d), got shape {arr.shape}")
        if arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValueError(f"need n >= 1 and d >= 1, got shape {arr.shape}")
        if not np.isfinite(arr).all():
            raise ValueError("point data contains NaN or infinite entries")
        self.data = arr

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def d(self) -> int:
        return self.data.shape[1]


def bin_point(point, h: float) -> GridIndex:
    """Host scalar helper, grid.py:62-75: floor(point/h) per axis."""
    h = check_bandwidth(h)
    p = np.asarray(point, dtype=np.float64)
    if p.ndim != 1:
        raise ValueError(f"point must be a flat vector, got shape {p.shape}")
    if not np.isfinite(p).all():
        raise ValueError("point has NaN or infinite coordinates")
    return tuple(int(math.floor(v / h)) for v in p.tolist())


def bin_points(data: np.ndarray, h: float) -> np.ndarray:
    """Host helper, grid.py:78-85 (the engine bins on device)."""
    h = check_bandwidth(h)
    q = np.floor(np.asarray(data, dtype=np.float64) / h)
    if q.size and np.abs(q).max() >= COORD_LIMIT:
        raise ValueError("cell coordinates exceed the supported integer lattice; "
                         "bandwidth is too small for this coordinate range")
    return q.astype(np.int64)


@dataclass
class CellTables:
    """Occupied-cell tables (grid.py:88-134): lexicographically sorted cells,
    counts >= 1 and coordinate sums; optional 3^d neighbour statistics."""

    cells: np.ndarray    # (k, d) int64
    counts: np.ndarray   # (k,) int64
    sums: np.ndarray     # (k, d) float64
    h: float
    n: int
    nbr_counts: np.ndarray | None = field(default=None, repr=False)
    nbr_sums: np.ndarray | None = field(default=None, repr=False)
    _cell_index: dict | None = field(default=None, repr=False)

    @property
    def d(self) -> int:
        return self.cells.shape[1]

    @property
    def k(self) -> int:
        return self.cells.shape[0]

    @property
    def index(self) -> dict:
        if self._cell_index is None:
            self._cell_index = {tuple(r): i for i, r in enumerate(self.cells.tolist())}
        return self._cell_index

    @property
    def count(self) -> dict:
        return {g: int(self.counts[i]) for g, i in self.index.items()}

    @property
    def sum(self) -> dict:
        return {g: self.sums[i].copy() for g, i in self.index.items()}

    def count_of(self, g) -> int:
        i = self.index.get(tuple(int(c) for c in g))
        return 0 if i is None else int(self.counts[i])


def _tables(points: PointSet, h: float, with_neighbours: bool) -> CellTables:
    h = check_bandwidth(h)
    L = _lib.load()
    ctx = _lib.context()
    y = points.data
    n, d = y.shape
    k = C.c_int64(0)
    _lib.check(L.gs_build_tables(ctx, _lib.ptr(y), n, d, h, 0, None, None, None, None, None,
                                 _lib.ref(k)))
    kk = int(k.value)
    cells = np.empty((kk, d), dtype=np.int64)
    counts = np.empty(kk, dtype=np.int64)
    sums = np.empty((kk, d), dtype=np.float64)
    nc = np.empty(kk, dtype=np.int64) if with_neighbours else None
    ns = np.empty((kk, d), dtype=np.float64) if with_neighbours else None
    _lib.check(L.gs_build_tables(ctx, _lib.ptr(y), n, d, h, kk, _lib.ptr(cells), _lib.ptr(counts),
                                 _lib.ptr(sums), _lib.ptr(nc), _lib.ptr(ns), _lib.ref(k)))
    return CellTables(cells=cells, counts=counts, sums=sums, h=h, n=n, nbr_counts=nc, nbr_sums=ns)


def build_cell_tables(points: PointSet, h: float, with_neighbours: bool = False) -> CellTables:
    """grid.py:193-196 on device: one pass, per-cell count and exact sum."""
    return _tables(points, h, with_neighbours)


def neighbor_stats(points: PointSet, h: float) -> CellTables:
    """Tables plus the 3^d neighbourhood count/sum of every occupied cell
    (grid.py:230-273, `_neighbor_stats_cells`), computed on device."""
    return _tables(points, h, True)


def neighbor_aggregate(tables: CellTables, g) -> tuple[int, np.ndarray]:
    """Scalar query over device-built tables (grid.py:211-227)."""
    g = tuple(int(c) for c in g)
    if len(g) != tables.d:
        raise ValueError(f"query cell has dimension {len(g)}, tables have {tables.d}")
    idx = tables.index
    total = 0
    acc = np.zeros(tables.d, dtype=np.float64)
    for v in itertools.product((-1, 0, 1), repeat=tables.d):
        r = idx.get(tuple(a + b for a, b in zip(g, v)))
        if r is not None:
            total += int(tables.counts[r])
            acc += tables.sums[r]
    return total, acc
