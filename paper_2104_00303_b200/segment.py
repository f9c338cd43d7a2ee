"""Image segmentation surface of the reference (`gridshift/segment.py`).

`segment_image` uploads the uint8 raster (3 B/pixel) and builds the fp64
(r, g, b[, x*s, y*s]) features inside the first engine kernel
(`gs_segment_image`), instead of shipping 24-40 B/pixel feature rows.
The features are bit-identical to `image_to_features` (segment.py:82-92).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .grid import PointSet
from .modeseek import ENGINES, Labeling, ShiftConfig, ShiftTrace, _finish

_MODES = ("rgb", "rgbxy")


@dataclass
class Image:
    """8-bit RGB raster, (height, width, 3) row-major (segment.py:28-48)."""

    pixels: np.ndarray

    def __post_init__(self):
        self.pixels = np.ascontiguousarray(self.pixels, dtype=np.uint8)
        if self.pixels.ndim != 3 or self.pixels.shape[2] != 3:
            raise ValueError(f"pixels must be (height, width, 3), got {self.pixels.shape}")
        if self.pixels.shape[0] < 1 or self.pixels.shape[1] < 1:
            raise ValueError("image must contain at least one pixel")

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def width(self) -> int:
        return self.pixels.shape[1]


@dataclass
class SegmentMap:
    """Per-pixel segment ids + mean colour per segment (segment.py:51-74)."""

    labels: np.ndarray
    k: int
    mean_colors: np.ndarray

    def __post_init__(self):
        self.labels = np.ascontiguousarray(self.labels, dtype=np.int64)
        if self.labels.ndim != 2:
            raise ValueError(f"labels must be 2-d, got shape {self.labels.shape}")
        self.mean_colors = np.asarray(self.mean_colors, dtype=np.float64)
        if self.mean_colors.shape != (self.k, 3):
            raise ValueError(f"mean_colors must be ({self.k}, 3), got {self.mean_colors.shape}")


def spatial_scale(img: Image) -> float:
    """segment.py:77-79."""
    return 255.0 / max(img.width, img.height)


def image_to_features(img: Image, mode: str = "rgb", scale: float | None = None) -> PointSet:
    """Host feature rows (segment.py:82-92); the engine path fuses this."""
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}, got {mode!r}")
    rgb = img.pixels.reshape(-1, 3).astype(np.float64)
    if mode == "rgb":
        return PointSet(rgb)
    s = spatial_scale(img) if scale is None else float(scale)
    ys, xs = np.divmod(np.arange(img.height * img.width), img.width)
    return PointSet(np.column_stack([rgb, xs * s, ys * s]))


def segment_pixels(img: Image, cfg: ShiftConfig, mode: str = "rgb",
                   scale: float | None = None) -> tuple[Labeling, ShiftTrace]:
    """Fused features + MeanShift++ on device (gs_segment_image)."""
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}, got {mode!r}")
    s = (spatial_scale(img) if scale is None else float(scale)) if mode == "rgbxy" else 0.0
    L = _lib.load()
    ctx = _lib.context()
    n = img.height * img.width
    d = 3 if mode == "rgb" else 5
    labels = np.empty(n, dtype=np.int64)
    mv = np.zeros(int(cfg.max_iters), dtype=np.float64)
    k, it, conv = C.c_int64(0), C.c_int32(0), C.c_int32(0)
    _lib.check(L.gs_segment_image(ctx, _lib.ptr(img.pixels), img.height, img.width,
                                  0 if mode == "rgb" else 1, s, float(cfg.h), cfg.resolve_eta(n),
                                  int(cfg.max_iters), _lib.ptr(labels), _lib.ref(k), _lib.ref(it),
                                  _lib.ptr(mv), _lib.ref(conv)))
    return _finish(ctx, labels, int(k.value), d, int(it.value), mv, conv.value)


def segment_image(img: Image, cfg: ShiftConfig, mode: str = "rgb", engine: str = "meanshiftpp",
                  scale: float | None = None):
    """segment.py:95-106: returns (SegmentMap, ShiftTrace)."""
    if engine not in ENGINES:
        raise ValueError(f"engine must be one of {sorted(ENGINES)}, got {engine!r}")
    labeling, trace = segment_pixels(img, cfg, mode, scale)
    # SegmentMap on device (segment.py:109-117): the labels come back in
    # raster order; the per-segment colour sums were accumulated on the GPU
    # next to the label delivery (gs_fetch_mean_colors), exact in integers
    mean = np.empty((labeling.k, 3), dtype=np.float64)
    _lib.check(_lib.load().gs_fetch_mean_colors(_lib.context(), _lib.ptr(mean), labeling.k))
    return SegmentMap(labels=labeling.labels.reshape(img.height, img.width), k=labeling.k,
                      mean_colors=mean), trace


def segment_map_from_labeling(img: Image, labeling: Labeling) -> SegmentMap:
    """segment.py:109-117 on the host, for labelings that did not come from
    segment_image (which gets the mean colours from the device)."""
    labels = labeling.labels.reshape(img.height, img.width)
    rgb = img.pixels.reshape(-1, 3).astype(np.float64)
    k = labeling.k
    cnt = np.bincount(labeling.labels, minlength=k).astype(np.float64)
    mean = np.column_stack([np.bincount(labeling.labels, weights=rgb[:, c], minlength=k) / cnt
                            for c in range(3)])
    return SegmentMap(labels=labels, k=k, mean_colors=mean)
