"""Exact-arithmetic model of the CUDA engine (test infrastructure).

Same algorithm as the reference (gridshift/grid.py + modeseek.py, restated
in oracle/gridshift_oracle.py), but with the engine's reductions:

  * per-cell and 3^d-neighbourhood coordinate sums are exact sums of the
    fixed-point images rint(y * 2^s_j), rounded once to fp64
    (gs_common.cuh: to_fixed / i128_to_double);
  * y' = S / C in fp64 (modeseek.py:109);
  * movement = exact sum of rint(norm * 2^(96-E)) rounded once;
  * modes = exact per-cluster sums / counts.

It reproduces the GPU results BIT FOR BIT (tests/test_gpu_exact.py), which
pins every device reduction; the distance between this model and the
reference's sequential-fp64 sums is then the reference's own rounding.
"""

from __future__ import annotations

import math

import numpy as np

from oracle import gridshift_oracle as O


class Params:
    """The engine's per-run constants (gs_engine.cu make_plan)."""

    def __init__(self, y0: np.ndarray, h: float):
        d = y0.shape[1]
        cells = np.floor(y0 / h)
        cmin, cmax = cells.min(axis=0), cells.max(axis=0)
        self.qexp = []
        span2 = 0.0
        for j in range(d):
            m = float(np.abs(y0[:, j]).max())
            e = math.frexp(m)[1] if m > 0 else 0
            self.qexp.append(max(-1000, min(1000, 62 - (e + 1))))
            ext = (cmax[j] - cmin[j]) + 5
            w = float(ext) * h
            span2 += w * w
        self.movement_exp = math.frexp(math.sqrt(span2) * 1.0000001 + 1e-300)[1]


def _fixed(y, s):
    return np.rint(np.ldexp(y, s)).astype(np.int64)


def _round(hi: np.ndarray, lo: np.ndarray, s: int) -> np.ndarray:
    """Correctly rounded fp64 of (hi * 2^32 + lo) * 2^-s (|result| < 2^85)."""
    carry = lo >> 32
    hi2 = hi + carry
    lo2 = lo & 0xFFFFFFFF
    return np.ldexp(hi2.astype(np.float64) * 4294967296.0 + lo2.astype(np.float64), -s)


def _group_sums(inverse: np.ndarray, k: int, vals: np.ndarray) -> np.ndarray:
    """Exact int64 sums of vals grouped by inverse (sort + reduceat)."""
    order = np.argsort(inverse, kind="stable")
    iv = inverse[order]
    starts = np.flatnonzero(np.r_[True, iv[1:] != iv[:-1]])
    out = np.zeros(k, dtype=np.int64)
    out[iv[starts]] = np.add.reduceat(vals[order], starts)
    return out


def _tables(y, h, P):
    cells = O.bin_cells(y, h)
    radix = O.mixed_radix(cells)
    keys, strides = radix
    ukeys, first, inverse, counts = np.unique(keys, return_index=True, return_inverse=True,
                                              return_counts=True)
    inverse = inverse.reshape(-1)
    k, d = ukeys.size, y.shape[1]
    hi = np.empty((k, d), dtype=np.int64)
    lo = np.empty((k, d), dtype=np.int64)
    for j in range(d):
        f = _fixed(y[:, j], P.qexp[j])
        hi[:, j] = _group_sums(inverse, k, f >> 32)
        lo[:, j] = _group_sums(inverse, k, f & 0xFFFFFFFF)
    return cells[first], ukeys, strides, counts.astype(np.int64), hi, lo, inverse


def _exact_sum_u(vals_hi: np.ndarray, vals_lo: np.ndarray) -> int:
    tot = 0
    for a in range(0, vals_hi.size, 1 << 14):
        tot += int(vals_hi[a:a + (1 << 14)].sum()) << 48
        tot += int(vals_lo[a:a + (1 << 14)].sum())
    return tot


def movement(y, y2, P) -> float:
    sq = (y2 - y) ** 2
    norm = np.sqrt(sq.sum(axis=1))
    a = np.ldexp(norm, 48 - P.movement_exp)
    ia = np.floor(a)
    hi = ia.astype(np.int64)
    lo = np.rint(np.ldexp(a - ia, 48)).astype(np.int64)
    return math.ldexp(float(_exact_sum_u(hi, lo)), P.movement_exp - 96)


def shift_once(y, h, P):
    cells, keys, strides, counts, hi, lo, inverse = _tables(y, h, P)
    k, d = hi.shape
    deltas = O.neighbour_offsets(d) @ strides
    nc = np.zeros(k, dtype=np.int64)
    nhi = np.zeros((k, d), dtype=np.int64)
    nlo = np.zeros((k, d), dtype=np.int64)
    for dl in deltas:
        q = keys + dl
        pos = np.minimum(np.searchsorted(keys, q), k - 1)
        hit = keys[pos] == q
        nc[hit] += counts[pos[hit]]
        nhi[hit] += hi[pos[hit]]
        nlo[hit] += lo[pos[hit]]
    tgt = np.empty((k, d))
    for j in range(d):
        tgt[:, j] = _round(nhi[:, j], nlo[:, j], P.qexp[j]) / nc.astype(np.float64)
    y2 = tgt[inverse]
    return y2, movement(y, y2, P), cells, counts


def extract(y, h, P):
    cells, keys, strides, counts, hi, lo, inverse = _tables(y, h, P)
    comp = O.components(cells)[inverse]
    ucomp, first_idx = np.unique(comp, return_index=True)
    rank = np.empty(ucomp.size, dtype=np.int64)
    rank[np.argsort(first_idx, kind="stable")] = np.arange(ucomp.size)
    labels = rank[np.searchsorted(ucomp, comp)]
    k, d = ucomp.size, y.shape[1]
    cnt = np.bincount(labels, minlength=k).astype(np.float64)
    modes = np.empty((k, d))
    for j in range(d):
        f = _fixed(y[:, j], P.qexp[j])
        modes[:, j] = _round(_group_sums(labels, k, f >> 32), _group_sums(labels, k, f & 0xFFFFFFFF),
                             P.qexp[j]) / cnt
    return labels, k, modes


def meanshiftpp(y0, h, eta=None, max_iters=300):
    y = np.ascontiguousarray(y0, dtype=np.float64)
    P = Params(y, h)
    thr = O.resolve_eta(eta, y.shape[0], h)
    hist, ks, fps = [], [], []
    converged = False
    from paper_2104_00303_b200 import workloads as W

    for _ in range(int(max_iters)):
        y2, mv, cells, counts = shift_once(y, h, P)
        ks.append(int(counts.size))
        fps.append(W.fingerprint(cells, counts))
        y = y2
        hist.append(mv)
        if mv < thr:
            converged = True
            break
    labels, k, modes = extract(y, h, P)
    return dict(labels=labels, k=k, modes=modes, iterations=len(hist),
                movement=np.asarray(hist), converged=converged, y=y, iter_k=ks, iter_fp=fps)
