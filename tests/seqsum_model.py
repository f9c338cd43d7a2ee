"""Sequential-sum model of the CUDA engine's reference-tracking table sums
(test infrastructure).

The reference accumulates every per-cell coordinate sum with np.bincount,
i.e. sequentially in point order starting from 0.0 (grid.py:186-187).
After the first iteration every point of a cell at t-1 sits at the same
position at t (modeseek.py:109), so most cells hold c copies of ONE value
v, and the reference's sum is fl(...fl(fl(0+v)+v)...+v), c additions.
That sum has a closed form per binade of the accumulator: while the
accumulator stays in [2^e, 2^(e+1)), adding v adds round(v / ulp) ulps
(ties to even make every addition after the first tie add an even number
of ulps), so the whole binade is one integer multiply-add; only the
addition that crosses into the next binade is done in fp64.  O(log c)
per cell instead of O(c), and bit-identical to the reference.

Cells whose points hold more than one distinct value (a group merging into
another) keep the engine's exact fixed-point sum rounded once; so does the
first table (distinct input values).

`seqsum_const` is the scalar/vector restatement the CUDA kernel follows
(gs_common.cuh seqsum_const); `meanshiftpp` is the whole-run model the GPU
is pinned to bit for bit.
"""

from __future__ import annotations

import math

import numpy as np

from oracle import gridshift_oracle as O

TWO53 = float(2 ** 53)


def seqsum_const(v: np.ndarray, c: np.ndarray) -> np.ndarray:
    """fl-sequential sum of c copies of v starting from 0.0 (vectorised).

    v float64, c int64 >= 1, same shape.  Bit-identical to
    np.add.accumulate(np.full(c, v))[-1] and to np.bincount's per-bin sum.
    """
    v = np.asarray(v, dtype=np.float64)
    c = np.asarray(c, dtype=np.int64)
    out = np.empty_like(v)
    sgn = np.sign(v)
    a = np.abs(v)
    s = a.copy()                   # first addition 0 + v is exact
    rem = c - 1
    live = (rem > 0) & (a > 0)
    while live.any():
        idx = np.flatnonzero(live)
        si, ai, ri = s[idx], a[idx], rem[idx]
        _, E = np.frexp(si)        # si = f * 2^E, f in [0.5, 1)
        ulp_e = E - 53
        m = np.ldexp(si, -ulp_e).astype(np.int64)          # exact, in [2^52, 2^53)
        x = np.ldexp(ai, -ulp_e)                            # a / ulp, exact scaling
        fl = np.floor(x)
        frac = x - fl
        fl = fl.astype(np.int64)
        tie = frac == 0.5
        delta = np.where(frac > 0.5, fl + 1, fl)
        # a tie adds fl or fl+1 so that the result is even; from then on the
        # accumulator is even and every tie addition adds fl rounded up to even
        first_tie = tie & (ri > 0)
        d1 = fl + ((m + fl) & 1)
        ok1 = first_tie & (m + d1 <= (1 << 53) - 1)
        m = np.where(ok1, m + d1, m)
        ri = np.where(ok1, ri - 1, ri)
        delta = np.where(tie, fl + (fl & 1), delta)
        lim = (1 << 53) - 1 - m
        k = np.where(delta > 0, np.minimum(ri, lim // np.maximum(delta, 1)), ri)
        k = np.where(tie & ~ok1, 0, k)
        m = m + k * delta
        ri = ri - k
        si = np.ldexp(m.astype(np.float64), ulp_e)
        # one real fp64 addition across the binade boundary (or the first
        # tie addition that would reach it)
        step = ri > 0
        si = np.where(step, si + ai, si)
        ri = np.where(step, ri - 1, ri)
        s[idx] = si
        rem[idx] = ri
        live[idx] = ri > 0
    out[:] = sgn * s
    return out


def _sequential(v: float, c: int) -> float:
    return float(np.add.accumulate(np.full(c, v))[-1])


def self_check(trials: int = 2000, seed: int = 0) -> None:
    rng = np.random.default_rng(seed)
    for t in range(trials):
        c = int(rng.integers(1, 5000))
        v = float(rng.normal(0, 10.0 ** rng.uniform(-3, 3)))
        if t % 5 == 0:   # values with few mantissa bits (ties)
            v = float(np.round(v * 64) / 64)
        got = float(seqsum_const(np.array([v]), np.array([c]))[0])
        want = _sequential(v, c)
        assert got == want or (math.isnan(got) and math.isnan(want)), (v, c, got, want)


# ------------------------------------------------------------------ model

def _exact_round(vals_by_cell: np.ndarray, inverse: np.ndarray, k: int) -> np.ndarray:
    """Correctly rounded per-cell sums (exact rational sum, one rounding)."""
    from fractions import Fraction  # noqa: F401  (documented alternative)

    order = np.argsort(inverse, kind="stable")
    iv = inverse[order]
    v = vals_by_cell[order]
    starts = np.flatnonzero(np.r_[True, iv[1:] != iv[:-1]])
    out = np.zeros(k)
    # math.fsum per cell: exactly rounded
    bounds = np.r_[starts, iv.size]
    for a, b in zip(bounds[:-1], bounds[1:]):
        out[iv[a]] = math.fsum(v[a:b])
    return out


def tables(y: np.ndarray, h: float, first: bool):
    """Per-cell (cells, keys, strides, counts, sums, inverse) with the
    engine's reference-tracking sums."""
    cells = O.bin_cells(y, h)
    keys, strides = O.mixed_radix(cells)
    ukeys, firsti, inverse, counts = np.unique(keys, return_index=True, return_inverse=True,
                                               return_counts=True)
    inverse = inverse.reshape(-1)
    k, d = ukeys.size, y.shape[1]
    sums = np.empty((k, d))
    if first:
        for j in range(d):
            sums[:, j] = _exact_round(y[:, j], inverse, k)
        return cells[firsti], ukeys, strides, counts, sums, inverse
    # one value per cell?  (min == max on every axis)
    uni = np.ones(k, dtype=bool)
    rep = y[firsti]
    for j in range(d):
        uni &= np.bincount(inverse, weights=(y[:, j] != rep[inverse, j]).astype(np.float64),
                           minlength=k) == 0
    for j in range(d):
        sums[:, j] = seqsum_const(rep[:, j], counts)
    mixed = np.flatnonzero(~uni)
    if mixed.size:
        sel = np.isin(inverse, mixed)
        sub_inv = np.searchsorted(mixed, inverse[sel])
        for j in range(d):
            sums[mixed, j] = _exact_round(y[sel, j], sub_inv, mixed.size)
    return cells[firsti], ukeys, strides, counts, sums, inverse


def shift_once(y, h, first):
    cells, keys, strides, counts, sums, inverse = tables(y, h, first)
    k, d = sums.shape
    deltas = O.neighbour_offsets(d) @ strides
    nc = np.zeros(k, dtype=np.int64)
    ns = np.zeros((k, d))
    for dl in deltas:          # sequential fp64 in offset order (grid.py:253-258)
        q = keys + dl
        pos = np.minimum(np.searchsorted(keys, q), k - 1)
        hit = keys[pos] == q
        nc[hit] += counts[pos[hit]]
        ns[hit] += sums[pos[hit]]
    y2 = ns[inverse] / nc[inverse, None].astype(np.float64)
    mv = float(np.sqrt(((y2 - y) ** 2).sum(axis=1)).sum())
    return y2, mv, cells, counts


def meanshiftpp(y0, h, eta=None, max_iters=300):
    from paper_2104_00303_b200 import workloads as W

    y = np.ascontiguousarray(y0, dtype=np.float64)
    thr = O.resolve_eta(eta, y.shape[0], h)
    hist, ks, fps = [], [], []
    converged = False
    for it in range(int(max_iters)):
        y2, mv, cells, counts = shift_once(y, h, it == 0)
        ks.append(int(counts.size))
        fps.append(W.fingerprint(cells, counts))
        y = y2
        hist.append(mv)
        if mv < thr:
            converged = True
            break
    r = O.extract(y, h)
    return dict(labels=r[0], k=r[1], modes=r[2], iterations=len(hist), movement=np.asarray(hist),
                converged=converged, y=y, iter_k=ks, iter_fp=fps)
