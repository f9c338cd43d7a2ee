"""Sequential-model restatement of the CUDA engine's DEFAULT sum order (test
infrastructure; the GPU is pinned to it bit for bit by
tests/test_gpu_parity.py::test_run_bitwise_vs_sequential_model).

Same algorithm as the reference (oracle/gridshift_oracle.py) with the
engine's default reductions (gs_refsum.cuh):

  * first table: exact fixed-point sums rounded once (tests/exact_model.py);
  * a cell that one source cell moved into: the reference's sequential sum
    of c copies of one value (seqsum_const: np.bincount's order, closed form);
  * a cell that several source cells moved into: model_fold32 -- the sources
    in ascending cell order, consumed in proportion inside each binade of the
    accumulator, single fp64 additions across the binade boundaries;
  * neighbourhood sums sequential in lexicographic offset order
    (grid.py:253-258); movement and modes exact (as in every sum order).

Dense lattice tables only (d <= 3): the engine orders a target's sources by
table slot, which is cell order there.
"""

from __future__ import annotations

import math
import struct

import numpy as np

from oracle import gridshift_oracle as O
from tests import exact_model as X
from tests.seqsum_model import seqsum_const

K_MAX_M = (1 << 53) - 1
K_DIRECT = 96


def _bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _butterfly(vals):
    """__shfl_xor_sync tree sum over 32 lanes (the value every lane ends with)."""
    a = list(vals) + [0.0] * (32 - len(vals))
    for o in (16, 8, 4, 2, 1):
        a = [a[i] + a[i ^ o] for i in range(32)]
    return a[0]


def model_fold32(cnt, val):
    """gs_refsum.cuh model_fold32: magnitudes val[a] with cnt[a] copies each,
    sources in ascending slot order (at most 32)."""
    m = len(cnt)
    rem = [int(c) for c in cnt]
    s = 0.0
    if sum(min(c, K_DIRECT + 1) for c in rem) <= K_DIRECT:
        while any(rem):
            live = [a for a in range(m) if rem[a] > 0]
            for a in live:
                s = val[a] if s == 0.0 else s + val[a]
            for a in live:
                rem[a] -= 1
        return s
    while any(rem):
        single, be = False, 0
        if s == 0.0:
            single = True
        else:
            sb = _bits(s)
            be = sb >> 52
            if be <= 1:
                single = True
            else:
                ue = be - 1075
                mi = (sb & ((1 << 52) - 1)) | (1 << 52)
                room = K_MAX_M - mi
                ia = [0] * m
                prod = [0.0] * m
                for a in range(m):
                    if rem[a]:
                        x = math.ldexp(val[a], -ue)
                        if x >= 2.0 ** 53:
                            ia[a] = 1 << 53
                        else:
                            fl = math.floor(x)
                            fr = x - fl
                            ia[a] = int(fl) + (1 if (fr > 0.5 or (fr == 0.5 and int(fl) & 1)) else 0)
                    prod[a] = float(rem[a]) * float(ia[a])
                totd = _butterfly(prod)
                if totd == 0.0:
                    break
                if totd <= float(room) * (1.0 - 2.0 ** -20):
                    mi += sum(r * i for r, i in zip(rem, ia))
                    s = math.ldexp(float(mi), ue)
                    break
                f = float(room) / totd * (1.0 - 2.0 ** -30)
                take = [0] * m
                for a in range(m):
                    if rem[a] and ia[a] < (1 << 53):
                        w = math.floor(f * float(rem[a]))
                        take[a] = 0 if w <= 0 else (rem[a] if w >= rem[a] else int(w))
                tk = sum(t * i for t, i in zip(take, ia))
                if tk > room:
                    take, tk = [0] * m, 0
                rem = [r - t for r, t in zip(rem, take)]
                mi += tk
                s = math.ldexp(float(mi), ue)
                single = True
        if single:
            for a in [a for a in range(m) if rem[a] > 0]:
                first = s == 0.0
                s = val[a] if first else s + val[a]
                rem[a] -= 1
                if first or (_bits(s) >> 52) != be:
                    break
    return s


def _neighbour_targets(keys, strides, counts, sums):
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
    return ns / nc[:, None].astype(np.float64)


def meanshiftpp(y0, h, eta=None, max_iters=300):
    from paper_2104_00303_b200 import workloads as W

    y = np.ascontiguousarray(y0, dtype=np.float64)
    n, d = y.shape
    if d > 3:
        raise ValueError("the sequential model orders sources by dense-table slot: d <= 3")
    P = X.Params(y, h)
    thr = O.resolve_eta(eta, n, h)
    cells, keys, strides, counts, hi, lo, inverse = X._tables(y, h, P)
    sums = np.empty((keys.size, d))
    for j in range(d):
        sums[:, j] = X._round(hi[:, j], lo[:, j], P.qexp[j])
    hist, ks, fps = [], [], []
    converged = False
    for _ in range(int(max_iters)):
        tgt = _neighbour_targets(keys, strides, counts, sums)
        y2 = tgt[inverse]
        hist.append(X.movement(y, y2, P))
        ks.append(int(counts.size))
        fps.append(W.fingerprint(cells, counts))
        y = y2
        if hist[-1] < thr:
            converged = True
            break
        # table t+1 from the cells of table t: every point of a cell moved to its target
        tcells = O.bin_cells(tgt, h)
        tkeys, strides = O.mixed_radix(tcells)
        ukeys, first, inv_src = np.unique(tkeys, return_index=True, return_inverse=True)
        inv_src = inv_src.reshape(-1)
        k2 = ukeys.size
        ncount = np.bincount(inv_src, weights=counts.astype(np.float64), minlength=k2).astype(np.int64)
        nsrc = np.bincount(inv_src, minlength=k2)
        nsums = np.empty((k2, d))
        single = nsrc[inv_src] == 1                      # per source: its target has one source
        tsel = inv_src[single]
        for j in range(d):
            nsums[tsel, j] = seqsum_const(tgt[single, j], counts[single])
        order = np.argsort(inv_src, kind="stable")       # sources by target, ascending source cell
        bounds = np.r_[0, np.cumsum(nsrc)]
        for t in np.flatnonzero(nsrc > 1):
            src = order[bounds[t]:bounds[t + 1]]
            for j in range(d):
                v = tgt[src, j]
                mag = model_fold32(counts[src].tolist(), np.abs(v).tolist())
                nsums[t, j] = -mag if (np.any(v < 0.0) and mag != 0.0) else mag
        cells, keys, counts, sums = tcells[first], ukeys, ncount, nsums
        inverse = inv_src[inverse]
    labels, k, modes = X.extract(y, h, P)
    return dict(labels=labels, k=k, modes=modes, iterations=len(hist), movement=np.asarray(hist),
                converged=converged, y=y, iter_k=ks, iter_fp=fps)
