"""MeanShift++ engine surface of the reference (`gridshift/modeseek.py`),
executed by the sm_100a kernels behind `libgridshift_cuda.so`.

Drop-in: `meanshiftpp(PointSet, ShiftConfig) -> (Labeling, ShiftTrace)` has
the reference signature (modeseek.py:125) and is what `ENGINES["meanshiftpp"]`
holds (modeseek.py:288).  `install()` swaps it into an importable reference
`gridshift` package so every caller there (segment_image, bench, CLI,
tracker) runs on the GPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import PointSet, check_bandwidth

_KERNELS = ("flat", "gaussian")
DEFAULT_MAX_ITERS = 300      # modeseek.py:42
ETA_SCALE = 1e-4             # modeseek.py:45


@dataclass
class ShiftConfig:
    """modeseek.py:48-74 (kernel only matters for the quadratic baseline,
    which this engine does not provide)."""

    h: float
    eta: float | None = None
    max_iters: int = DEFAULT_MAX_ITERS
    kernel: str = "flat"

    def __post_init__(self):
        check_bandwidth(self.h)
        if self.eta is not None and (not np.isfinite(self.eta) or self.eta <= 0):
            raise ValueError(f"eta must be positive and finite, got {self.eta}")
        if int(self.max_iters) != self.max_iters or self.max_iters < 1:
            raise ValueError(f"max_iters must be a positive integer, got {self.max_iters}")
        if self.kernel not in _KERNELS:
            raise ValueError(f"kernel must be one of {_KERNELS}, got {self.kernel!r}")

    def resolve_eta(self, n: int) -> float:
        return float(self.eta) if self.eta is not None else ETA_SCALE * n * self.h


@dataclass
class Labeling:
    """modeseek.py:77-91."""

    labels: np.ndarray
    k: int
    modes: np.ndarray

    def __post_init__(self):
        self.labels = np.ascontiguousarray(self.labels, dtype=np.int64)
        self.modes = np.ascontiguousarray(self.modes, dtype=np.float64)
        if self.k < 1 or self.modes.shape[0] != self.k:
            raise ValueError(f"expected {self.k} mode rows, got {self.modes.shape}")
        if self.labels.min() != 0 or self.labels.max() != self.k - 1:
            raise ValueError("labels must cover [0, k) densely")

    @classmethod
    def _from_engine(cls, labels, k, modes, d):
        """Engine results are dense in [0, k) by construction (first-appearance
        ranks of every component; checked by the GPU tests), so skip the O(n)
        host-side re-validation of user-built Labelings (2 passes over 800 MB
        at n = 1e8)."""
        obj = cls.__new__(cls)
        obj.labels = np.ascontiguousarray(labels, dtype=np.int64)
        obj.modes = np.ascontiguousarray(modes, dtype=np.float64)
        obj.k = int(k)
        if obj.k < 1 or obj.modes.shape != (obj.k, int(d)):
            raise RuntimeError(f"engine returned malformed modes {obj.modes.shape}, expected ({obj.k}, {d})")
        return obj


@dataclass
class ShiftTrace:
    """modeseek.py:94-100, plus per-iteration occupied-cell counts and
    (cells, counts) fingerprints recorded on device."""

    iterations: int
    total_movement_per_iter: np.ndarray = field(repr=False)
    converged: bool = False
    cells_per_iter: np.ndarray | None = field(default=None, repr=False)
    fingerprint_per_iter: np.ndarray | None = field(default=None, repr=False)


def _fetch(ctx, k: int, d: int, iters: int):
    L = _lib.load()
    modes = np.empty((k, d), dtype=np.float64)
    _lib.check(L.gs_fetch_modes(ctx, _lib.ptr(modes), k))
    kk = np.empty(iters, dtype=np.int64)
    fp = np.empty(iters, dtype=np.uint64)
    _lib.check(L.gs_fetch_trace(ctx, _lib.ptr(kk), _lib.ptr(fp), iters))
    return modes, kk, fp


def _finish(ctx, labels, k, d, iters, mv, conv):
    modes, kk, fp = _fetch(ctx, k, d, iters)
    lab = Labeling._from_engine(labels, k, modes, d)
    tr = ShiftTrace(iterations=iters, total_movement_per_iter=mv[:iters].copy(),
                    converged=bool(conv), cells_per_iter=kk, fingerprint_per_iter=fp)
    return lab, tr


def host_labels(labels_out, n: int) -> np.ndarray:
    """The (n,) int64 host label buffer the C ABI writes n entries into:
    a fresh array, or the caller's after checking shape, dtype and layout
    (the engine's streaming-store expansion trusts it)."""
    if labels_out is None:
        return np.empty(n, dtype=np.int64)
    if (not isinstance(labels_out, np.ndarray) or labels_out.shape != (n,)
            or labels_out.dtype != np.int64 or not labels_out.flags.c_contiguous
            or not labels_out.flags.writeable):
        raise ValueError(f"labels_out must be a writeable C-contiguous ({n},) int64 array")
    return labels_out


def device_labels(labels_out, n: int, x):
    """The (n,) int64 CUDA label tensor for the device entry points:
    allocated on x's device, or the caller's after checking numel, dtype,
    contiguity and device."""
    import torch

    if labels_out is None:
        return torch.empty(n, dtype=torch.int64, device=x.device)
    if (not isinstance(labels_out, torch.Tensor) or labels_out.numel() != n
            or labels_out.dtype != torch.int64 or not labels_out.is_contiguous()
            or labels_out.device != x.device):
        raise ValueError(f"labels_out must be a contiguous int64 tensor of {n} elements on {x.device}")
    return labels_out


SUM_ORDERS = {"reference": _lib.GS_SUMS_REFERENCE, "exact": _lib.GS_SUMS_EXACT,
              "seqmodel": _lib.GS_SUMS_SEQMODEL}
DEFAULT_SUM_ORDER = "seqmodel"


def set_sum_order(order: str, device: int | None = None) -> None:
    """Summation order of this thread's engine context.

    "seqmodel" (default): the reference's sequential fp64 sums
    (np.bincount, grid.py:186-187) without the point order -- a cell holding
    c copies of one value gets the reference's sum bit for bit (closed form
    per binade), a cell that received several source cells folds them
    interleaved proportionally (no sort); neighbourhood sums in the
    reference's lexicographic offset order (grid.py:253-258).  Cells, counts
    and labels equal the reference's, modes within 1e-9*h on every
    configuration; assumes the points of a mixed cell
    are well mixed in index order (for 1e8 spatially sorted rows the modes
    can drift ~1e-8*h from the reference's, like the exact order's).
    "reference": additionally every mixed cell is summed in point-index
    order -- iterates equal the reference's bit for bit (about 2x slower).
    "exact": order-independent exact fixed-point sums rounded once (what the
    row-sharded multi-GPU path computes, independent of the split)."""
    if order not in SUM_ORDERS:
        raise ValueError(f"sum order must be one of {sorted(SUM_ORDERS)}, got {order!r}")
    _lib.check(_lib.load().gs_ctx_set_option(_lib.context(device), _lib.GS_OPT_SUMS, SUM_ORDERS[order]))


class sum_order:
    """Context manager: `with sum_order("exact"): ...` (this thread)."""

    def __init__(self, order: str, device: int | None = None):
        self.order, self.device = order, device

    def __enter__(self):
        set_sum_order(self.order, self.device)
        return self

    def __exit__(self, *exc):
        set_sum_order(DEFAULT_SUM_ORDER, self.device)


def meanshiftpp(points: PointSet, cfg: ShiftConfig, labels_out: np.ndarray | None = None
                ) -> tuple[Labeling, ShiftTrace]:
    """modeseek.py:125-146 on the B200: device-resident loop until the
    summed movement drops below eta (the converging step applied) or
    max_iters, then device-side cluster extraction.  `labels_out` may be a
    preallocated (n,) int64 array (e.g. pinned host memory)."""
    if not isinstance(points, PointSet):
        points = PointSet(points)
    L = _lib.load()
    ctx = _lib.context()
    y = points.data
    n, d = y.shape
    eta = cfg.resolve_eta(n)
    labels = host_labels(labels_out, n)
    mv = np.zeros(int(cfg.max_iters), dtype=np.float64)
    k, it, conv = C.c_int64(0), C.c_int32(0), C.c_int32(0)
    _lib.check(L.gs_meanshiftpp(ctx, _lib.ptr(y), n, d, float(cfg.h), eta, int(cfg.max_iters),
                                _lib.ptr(labels), _lib.ref(k), _lib.ref(it), _lib.ptr(mv),
                                _lib.ref(conv)))
    return _finish(ctx, labels, int(k.value), d, int(it.value), mv, conv.value)


def meanshiftpp_points(x: np.ndarray, cfg: ShiftConfig, labels_out: np.ndarray | None = None
                       ) -> tuple[Labeling, ShiftTrace]:
    """meanshiftpp on a raw host (n, d) array of float32 or float64 without
    building a PointSet: float32 rows cross PCIe as float32 and are upcast on
    device -- bit-identical to PointSet's host upcast (grid.py:43) at half
    the transfer.  Validation (finite, n, d >= 1) happens on device."""
    x = np.asarray(x)
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    x = np.ascontiguousarray(x)
    if x.ndim != 2:
        raise ValueError(f"point data must be 2-d (n, d), got shape {x.shape}")
    L = _lib.load()
    ctx = _lib.context()
    n, d = x.shape
    eta = cfg.resolve_eta(n)
    labels = host_labels(labels_out, n)
    mv = np.zeros(int(cfg.max_iters), dtype=np.float64)
    k, it, conv = C.c_int64(0), C.c_int32(0), C.c_int32(0)
    dt = _lib.GS_DTYPE_F32 if x.dtype == np.float32 else _lib.GS_DTYPE_F64
    _lib.check(L.gs_meanshiftpp_host(ctx, _lib.ptr(x), dt, n, d, float(cfg.h), eta, int(cfg.max_iters),
                                     _lib.ptr(labels), _lib.ref(k), _lib.ref(it), _lib.ptr(mv), _lib.ref(conv)))
    return _finish(ctx, labels, int(k.value), d, int(it.value), mv, conv.value)


def meanshiftpp_device(x, cfg: ShiftConfig, labels_out=None, stream=None, collapsed: bool = False):
    """Device-resident entry: `x` is a CUDA tensor (n, d) float64 or float32
    (anything exposing data_ptr()).  Labels are written into `labels_out`
    (CUDA int64 tensor, allocated if None).  Returns (labels_out, k, iters,
    movement, converged); modes via `last_modes()`.  collapsed=True runs
    iterations t >= 1 per run of identical points (bit-identical
    results, not a per-point workload)."""
    import torch

    L = _lib.load()
    dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
    ctx = _lib.context(dev)
    n, d = x.shape
    if not x.is_contiguous():
        raise ValueError("device point data must be C-contiguous")
    dtype = {torch.float64: _lib.GS_DTYPE_F64, torch.float32: _lib.GS_DTYPE_F32}.get(x.dtype)
    if dtype is None:
        raise ValueError("device point data must be float64 or float32")
    labels_out = device_labels(labels_out, n, x)
    eta = cfg.resolve_eta(n)
    mv = np.zeros(int(cfg.max_iters), dtype=np.float64)
    k, it, conv = C.c_int64(0), C.c_int32(0), C.c_int32(0)
    s = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(L.gs_ctx_set_option(ctx, _lib.GS_OPT_COLLAPSED, 1 if collapsed else 0))
    try:
        _lib.check(L.gs_meanshiftpp_device(ctx, C.c_void_p(x.data_ptr()), dtype, n, d, float(cfg.h),
                                           eta, int(cfg.max_iters), C.c_void_p(labels_out.data_ptr()),
                                           _lib.ref(k), _lib.ref(it), _lib.ptr(mv), _lib.ref(conv),
                                           C.c_void_p(s)))
    finally:
        _lib.check(L.gs_ctx_set_option(ctx, _lib.GS_OPT_COLLAPSED, 0))
    return labels_out, int(k.value), int(it.value), mv[: it.value].copy(), bool(conv.value)


def last_iterate(n: int, d: int, device: int | None = None) -> np.ndarray:
    """Final iterate (n, d) of this thread's last per-point run, original
    point order (test observability: the trajectory check against the
    reference/oracle bit for bit)."""
    y = np.empty((n, d), dtype=np.float64)
    _lib.check(_lib.load().gs_fetch_iterate(_lib.context(device), _lib.ptr(y), n))
    return y


def last_refsum_stats(iterations: int, device: int | None = None) -> np.ndarray:
    """Reference-order sum counters of this thread's last run, one row per
    table (row 0 = first table): segments folded in index order, long
    segments taking the global sort, their points, longest segment,
    recomputed single-source closed forms."""
    out = np.zeros((iterations + 1, 5), dtype=np.uint32)
    _lib.check(_lib.load().gs_fetch_refsum_stats(_lib.context(device), _lib.ptr(out), iterations + 1))
    return out


def last_modes(k: int, d: int, device: int | None = None) -> np.ndarray:
    modes = np.empty((k, d), dtype=np.float64)
    _lib.check(_lib.load().gs_fetch_modes(_lib.context(device), _lib.ptr(modes), k))
    return modes


def meanshiftpp_step(points: PointSet, cfg: ShiftConfig) -> tuple[PointSet, float]:
    """modeseek.py:114-122: one grid-neighbourhood mean update on device."""
    L = _lib.load()
    ctx = _lib.context()
    y = points.data
    n, d = y.shape
    out = np.empty_like(y)
    mv = C.c_double(0.0)
    _lib.check(L.gs_shift_step(ctx, _lib.ptr(y), n, d, float(cfg.h), _lib.ptr(out), _lib.ref(mv)))
    return PointSet(out), float(mv.value)


def extract_clusters(converged: PointSet, h: float) -> Labeling:
    """modeseek.py:275-285 on device: bin at h, union-find over Chebyshev
    adjacent occupied cells, first-appearance labels, mean modes."""
    h = check_bandwidth(h)
    L = _lib.load()
    ctx = _lib.context()
    y = converged.data
    n, d = y.shape
    labels = np.empty(n, dtype=np.int64)
    k = C.c_int64(0)
    _lib.check(L.gs_extract_clusters(ctx, _lib.ptr(y), n, d, h, _lib.ptr(labels), _lib.ref(k)))
    modes = np.empty((int(k.value), d), dtype=np.float64)
    _lib.check(L.gs_fetch_modes(ctx, _lib.ptr(modes), int(k.value)))
    return Labeling(labels=labels, k=int(k.value), modes=modes)


ENGINES = {"meanshiftpp": meanshiftpp}


def install(gridshift_module=None) -> None:
    """Register this engine in a reference `gridshift` installation.

    Patched (the reference's drop-in surfaces):
    ENGINES["meanshiftpp"] (modeseek.py:288, read by segment_image, bench
    and the CLI) and the module attributes `meanshiftpp`, `meanshiftpp_step`
    and `extract_clusters` of gridshift.modeseek (modeseek.py:114,125,275),
    plus track.py's direct import of meanshiftpp (track.py:22).  Callers
    that import these names AFTER install() (e.g. the reference's own test
    modules) get the CUDA engine; results come back as the reference's own
    Labeling / ShiftTrace / PointSet objects."""
    import importlib

    gs = gridshift_module or importlib.import_module("gridshift")
    ms = importlib.import_module(gs.__name__ + ".modeseek")
    rgrid = importlib.import_module(gs.__name__ + ".grid")

    def engine(points, cfg):
        lab, tr = meanshiftpp(PointSet(points.data), ShiftConfig(cfg.h, cfg.eta, cfg.max_iters))
        return (ms.Labeling(labels=lab.labels, k=lab.k, modes=lab.modes),
                ms.ShiftTrace(iterations=tr.iterations,
                              total_movement_per_iter=tr.total_movement_per_iter,
                              converged=tr.converged))

    def step(points, cfg):
        moved, mv = meanshiftpp_step(PointSet(points.data), ShiftConfig(cfg.h, cfg.eta, cfg.max_iters))
        return rgrid.PointSet(moved.data), mv

    def extract(converged, h):
        lab = extract_clusters(PointSet(converged.data), h)
        return ms.Labeling(labels=lab.labels, k=lab.k, modes=lab.modes)

    engine.__gridshift_b200__ = step.__gridshift_b200__ = extract.__gridshift_b200__ = True
    ms.ENGINES["meanshiftpp"] = engine
    ms.meanshiftpp = engine
    ms.meanshiftpp_step = step
    ms.extract_clusters = extract
    for sub in ("track", "segment", "bench", "cli"):
        try:
            mod = importlib.import_module(gs.__name__ + "." + sub)
        except ImportError:
            continue
        if hasattr(mod, "meanshiftpp"):
            mod.meanshiftpp = engine
