"""numpy backend for paper_2104_00303_b200.sharded (test infrastructure).

Mirrors the CUDA shard operations with the engine's exact integer
arithmetic (tests/exact_model.py): dense lattice table over the global box,
first table merged by the driver's all-reduce, later tables derived per
cell, shift of the local rows, 4-limb movement, per-root first-appearance
minima.  Lets the world-size-2 gloo test run the real driver on CPU.
"""

from __future__ import annotations

import itertools
import math

import numpy as np
import torch

from tests import exact_model as X
from paper_2104_00303_b200 import workloads as W

BIG = np.iinfo(np.int64).max


class NumpyShard:
    def __init__(self, x_local: np.ndarray):
        self.y = np.ascontiguousarray(x_local, dtype=np.float64)
        self.done = False
        self.iters = 0
        self.hist, self.ks, self.fps = [], [], []

    def new(self, count, kind):
        return torch.zeros(int(count), dtype={"i64": torch.int64, "f64": torch.float64}[kind])

    def init(self, d, h):
        self.d, self.h = d, float(h)
        n = self.y.shape[0]
        if n == 0:
            return (np.full(d, BIG, np.int64), np.full(d, -BIG - 1, np.int64), np.zeros(d), 0)
        cells = np.floor(self.y / self.h).astype(np.int64)
        return cells.min(axis=0), cells.max(axis=0), np.abs(self.y).max(axis=0), 0

    # -- lattice ---------------------------------------------------------
    def plan(self, cmin, cmax, amax, flags, n_total, max_iters):
        d, h = self.d, self.h
        self.qexp = []
        span2 = 0.0
        for j in range(d):
            m = float(amax[j])
            e = math.frexp(m)[1] if m > 0 else 0
            self.qexp.append(max(-1000, min(1000, 62 - (e + 1))))
            w = float(int(cmax[j]) - int(cmin[j]) + 5) * h
            span2 += w * w
        self.mexp = math.frexp(math.sqrt(span2) * 1.0000001 + 1e-300)[1]
        self.base = np.asarray(cmin, np.int64) - 2
        ext = (np.asarray(cmax, np.int64) - np.asarray(cmin, np.int64) + 5).tolist()
        self.strides = np.ones(d, np.int64)
        for j in range(d - 2, -1, -1):
            self.strides[j] = self.strides[j + 1] * ext[j + 1]
        self.nkeys = int(np.prod(ext))
        self.table = self._hist(self.y)
        return self.nkeys * (1 + 2 * d)

    def _keys(self, pts):
        cells = np.floor(pts / self.h).astype(np.int64)
        return (cells - self.base) @ self.strides

    def _hist(self, pts):
        d = self.d
        tab = np.zeros((self.nkeys, 1 + 2 * d), np.int64)
        if len(pts):
            k = self._keys(pts)
            np.add.at(tab[:, 0], k, 1)
            for j in range(d):
                f = X._fixed(pts[:, j], self.qexp[j])
                np.add.at(tab[:, 1 + j], k, f >> 32)
                np.add.at(tab[:, 1 + d + j], k, f & 0xFFFFFFFF)
        return tab

    def table_io(self, buf, to_device_table):
        if to_device_table:
            self.table = buf.numpy().reshape(self.nkeys, 1 + 2 * self.d).copy()
        else:
            buf.copy_(torch.from_numpy(self.table.ravel()))

    def _targets(self):
        d = self.d
        occ = np.flatnonzero(self.table[:, 0])
        deltas = [int(np.dot(v, self.strides)) for v in itertools.product((-1, 0, 1), repeat=d)]
        cnt = np.zeros(occ.size, np.int64)
        hi = np.zeros((occ.size, d), np.int64)
        lo = np.zeros((occ.size, d), np.int64)
        for dl in deltas:
            nb = self.table[occ + dl]
            cnt += nb[:, 0]
            hi += nb[:, 1:1 + d]
            lo += nb[:, 1 + d:]
        tgt = np.empty((occ.size, d))
        for j in range(d):
            tgt[:, j] = X._round(hi[:, j], lo[:, j], self.qexp[j]) / cnt.astype(np.float64)
        return occ, tgt

    def _cells_of(self, slots):
        d = self.d
        ext0 = self.nkeys // int(self.strides[0])
        out = np.empty((slots.size, d), np.int64)
        for j in range(d):
            e = ext0 if j == 0 else int(self.strides[j - 1] // self.strides[j])
            out[:, j] = (slots // self.strides[j]) % e + self.base[j]
        return out

    def iterate(self, t, limbs):
        if self.done:
            return
        d = self.d
        occ, tgt = self._targets()
        self.ks.append(int(occ.size))
        self.fps.append(W.fingerprint(self._cells_of(occ), self.table[occ, 0]))
        slot_of = np.full(self.nkeys, -1, np.int64)
        slot_of[occ] = np.arange(occ.size)
        y2 = tgt[slot_of[self._keys(self.y)]] if len(self.y) else self.y.copy()
        # movement: exact 128-bit fixed point, split into 32-bit limbs
        tot = 0
        if len(self.y):
            norm = np.sqrt(((y2 - self.y) ** 2).sum(axis=1))
            a = np.ldexp(norm, 48 - self.mexp)
            ia = np.floor(a)
            tot = X._exact_sum_u(ia.astype(np.int64), np.rint(np.ldexp(a - ia, 48)).astype(np.int64))
        limbs.copy_(torch.tensor([(tot >> (32 * i)) & 0xFFFFFFFF for i in range(4)], dtype=torch.int64))
        # derived next table (k_derive): count_c * fixed(target_c) at key(target_c)
        nxt = np.zeros_like(self.table)
        tk = self._keys(tgt)
        c = self.table[occ, 0]
        np.add.at(nxt[:, 0], tk, c)
        for j in range(d):
            f = X._fixed(tgt[:, j], self.qexp[j])
            np.add.at(nxt[:, 1 + j], tk, (f >> 32) * c)
            np.add.at(nxt[:, 1 + d + j], tk, (f & 0xFFFFFFFF) * c)
        self.table = nxt
        self.y = y2

    def converge(self, t, limbs, eta):
        if self.done:
            return
        tot = sum(int(v) << (32 * i) for i, v in enumerate(limbs.tolist()))
        mv = math.ldexp(float(tot), self.mexp - 96)
        self.hist.append(mv)
        self.iters = t + 1
        if mv < eta:
            self.done = True

    def status(self):
        return self.done, self.iters

    def components(self, offset, minima):
        from oracle import gridshift_oracle as O

        occ = np.flatnonzero(self.table[:, 0])
        comp = O.components(self._cells_of(occ))       # root row per cell (rows in key order)
        self.root_slot = np.full(self.nkeys, -1, np.int64)
        self.root_slot[occ] = occ[comp]
        self.occ = occ
        mins = np.full(self.nkeys, BIG, np.int64)
        if len(self.y):
            r = self.root_slot[self._keys(self.y)]
            np.minimum.at(mins, r, offset + np.arange(len(self.y)))
        minima.copy_(torch.from_numpy(mins))

    def finish(self, minima, labels, max_iters):
        d = self.d
        mins = minima.numpy()
        roots = np.unique(self.root_slot[self.occ])
        order = np.argsort(mins[roots], kind="stable")
        rank = np.empty(self.nkeys, np.int64)
        rank[roots[order]] = np.arange(roots.size)
        if len(self.y):
            labels.copy_(torch.from_numpy(rank[self.root_slot[self._keys(self.y)]]))
        k = roots.size
        cnt = np.zeros(k, np.int64)
        hi = np.zeros((k, d), np.int64)
        lo = np.zeros((k, d), np.int64)
        lab = rank[self.root_slot[self.occ]]
        np.add.at(cnt, lab, self.table[self.occ, 0])
        for j in range(d):
            np.add.at(hi[:, j], lab, self.table[self.occ, 1 + j])
            np.add.at(lo[:, j], lab, self.table[self.occ, 1 + d + j])
        self._modes = np.stack([X._round(hi[:, j], lo[:, j], self.qexp[j]) / cnt.astype(np.float64)
                                for j in range(d)], axis=1)
        return k, self.iters, np.asarray(self.hist), self.done

    def modes(self, k, d):
        return self._modes

    def trace(self, iters):
        return np.asarray(self.ks[:iters], np.int64), np.asarray(self.fps[:iters], np.uint64)
