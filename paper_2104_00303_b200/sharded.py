"""Row-sharded MeanShift++ over one process per GPU (cfg4-style strong
scaling), collectives through ``torch.distributed`` (NCCL on GPUs).

The reference is single-process; its spec allows "sharding points and
merging partial tables".  Because every
point of a cell moves to exactly that cell's target, the table of iteration
t+1 is a function of the table of iteration t alone (k_derive).  So only
the FIRST table is merged -- an integer all-reduce of the fixed-point table
words, exact and identical on every rank -- and each later table is derived
identically on every rank.  Per iteration the ranks exchange only the
movement (4 int64 limbs of an exact 128-bit sum); at the end one MIN
all-reduce gives the global first-appearance numbering.  Results equal the
single-GPU engine bit for bit, in the default sum order (the sequential
model of the reference's per-cell sums is a function of the merged cell
table only, so every rank computes the same sums) and in the exact order;
a context set to the reference order runs the default here (the point-index
order of a mixed cell spans ranks).

The per-rank work goes through a backend (default: the CUDA C ABI); tests
inject a numpy backend to cover this driver with gloo on CPU.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .modeseek import Labeling, ShiftConfig, ShiftTrace


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row range of `rank` (rows are pre-shuffled)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class CudaShard:
    """Per-rank engine operations through libgridshift_cuda.so."""

    def __init__(self, x_local):
        import torch

        self.torch = torch
        self.x = x_local
        self.dev = x_local.device
        self.ctx = _lib.context(self.dev.index)
        self.L = _lib.load()

    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.dev).cuda_stream)

    def new(self, count: int, kind: str):
        dt = {"i64": self.torch.int64, "f64": self.torch.float64}[kind]
        return self.torch.zeros(int(count), dtype=dt, device=self.dev)

    def init(self, d: int, h: float):
        t = self.torch
        dtype = {t.float64: _lib.GS_DTYPE_F64, t.float32: _lib.GS_DTYPE_F32}.get(self.x.dtype)
        if dtype is None:
            raise ValueError("device point data must be float64 or float32")
        cmin = np.zeros(d, dtype=np.int64)
        cmax = np.zeros(d, dtype=np.int64)
        amax = np.zeros(d, dtype=np.float64)
        flags = C.c_int32(0)
        _lib.check(self.L.gs_shard_init(self.ctx, C.c_void_p(self.x.data_ptr()), dtype, self.x.shape[0], d,
                                        float(h), self._stream(), _lib.ptr(cmin), _lib.ptr(cmax),
                                        _lib.ptr(amax), _lib.ref(flags)))
        return cmin, cmax, amax, int(flags.value)

    def plan(self, cmin, cmax, amax, flags, n_total, max_iters):
        words = C.c_int64(0)
        _lib.check(self.L.gs_shard_plan(self.ctx, _lib.ptr(cmin), _lib.ptr(cmax), _lib.ptr(amax), int(flags),
                                        int(n_total), int(max_iters), self._stream(), _lib.ref(words)))
        return int(words.value)

    def table_io(self, buf, to_device_table: bool):
        _lib.check(self.L.gs_shard_table_io(self.ctx, C.c_void_p(buf.data_ptr()), 1 if to_device_table else 0,
                                            self._stream()))

    def iterate(self, t, limbs):
        _lib.check(self.L.gs_shard_iterate(self.ctx, int(t), C.c_void_p(limbs.data_ptr()), self._stream()))

    def converge(self, t, limbs, eta):
        _lib.check(self.L.gs_shard_converge(self.ctx, int(t), C.c_void_p(limbs.data_ptr()), float(eta),
                                            self._stream()))

    def status(self):
        done, iters = C.c_int32(0), C.c_int32(0)
        _lib.check(self.L.gs_shard_status(self.ctx, _lib.ref(done), _lib.ref(iters), self._stream()))
        return bool(done.value), int(iters.value)

    def components(self, offset, minima):
        slots = C.c_int64(0)
        _lib.check(self.L.gs_shard_components(self.ctx, int(offset), C.c_void_p(minima.data_ptr()),
                                              self._stream(), _lib.ref(slots)))

    def finish(self, minima, labels, max_iters):
        k, it, conv = C.c_int64(0), C.c_int32(0), C.c_int32(0)
        mv = np.zeros(int(max_iters))
        _lib.check(self.L.gs_shard_finish(self.ctx, C.c_void_p(minima.data_ptr()), C.c_void_p(labels.data_ptr()),
                                          self._stream(), _lib.ref(k), _lib.ref(it), _lib.ptr(mv),
                                          _lib.ref(conv)))
        return int(k.value), int(it.value), mv[: it.value].copy(), bool(conv.value)

    def modes(self, k, d):
        m = np.empty((k, d))
        _lib.check(self.L.gs_fetch_modes(self.ctx, _lib.ptr(m), k))
        return m

    def trace(self, iters):
        kk = np.empty(iters, dtype=np.int64)
        fp = np.empty(iters, dtype=np.uint64)
        _lib.check(self.L.gs_fetch_trace(self.ctx, _lib.ptr(kk), _lib.ptr(fp), iters))
        return kk, fp


def _allreduce(dist, buf, op, group):
    dist.all_reduce(buf, op=op, group=group)
    return buf


def meanshiftpp_sharded(x_local, cfg: ShiftConfig, labels_out=None, n_total: int | None = None,
                        group=None, backend=None, chunk0: int = 4, return_result: bool = False):
    """One MeanShift++ run over the row shards of all ranks of `group`.

    x_local: this rank's rows, (n_local, d) (CUDA tensor for the default
    backend).  labels_out: (n_local,) int64 buffer on the backend's device
    (allocated if None) -- receives the labels of the local rows, numbered
    by first appearance in the GLOBAL row order (ranks hold consecutive row
    ranges in rank order).  Returns the iteration count, or
    (Labeling of the local rows, ShiftTrace) with return_result=True.
    """
    import torch
    import torch.distributed as dist

    be = backend or CudaShard(x_local)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n_local, d = int(x_local.shape[0]), int(x_local.shape[1])
    sizes = be.new(world, "i64")
    sizes[rank] = n_local
    _allreduce(dist, sizes, dist.ReduceOp.SUM, group)
    sizes = sizes.cpu().numpy()
    offset = int(sizes[:rank].sum())
    total = int(sizes.sum())
    if n_total is not None and int(n_total) != total:
        raise ValueError(f"n_total={n_total} but the shards hold {total} rows")
    # 1. global lattice box / quantisation: MIN/MAX of the local statistics
    cmin, cmax, amax, flags = be.init(d, cfg.h)
    lo = be.new(d, "i64")
    lo.copy_(torch.from_numpy(cmin))
    hi = be.new(d, "i64")
    hi.copy_(torch.from_numpy(cmax))
    am = be.new(d, "f64")
    am.copy_(torch.from_numpy(amax))
    fl = be.new(8, "i64")
    fl.copy_(torch.tensor([(flags >> b) & 1 for b in range(8)], dtype=torch.int64))
    _allreduce(dist, lo, dist.ReduceOp.MIN, group)
    _allreduce(dist, hi, dist.ReduceOp.MAX, group)
    _allreduce(dist, am, dist.ReduceOp.MAX, group)
    _allreduce(dist, fl, dist.ReduceOp.MAX, group)
    gflags = int(sum(int(v) << b for b, v in enumerate(fl.cpu().tolist())))
    words = be.plan(lo.cpu().numpy(), hi.cpu().numpy(), am.cpu().numpy(), gflags, total, cfg.max_iters)
    # 2. the only table merge: exact integer SUM of the first tables
    table = be.new(words, "i64")
    be.table_io(table, False)
    _allreduce(dist, table, dist.ReduceOp.SUM, group)
    be.table_io(table, True)
    del table
    # 3. device-driven iterations; only the 4-limb movement crosses ranks
    eta = cfg.resolve_eta(total)
    limbs = be.new(4, "i64")
    t, chunk = 0, chunk0
    while t < cfg.max_iters:
        for _ in range(min(chunk, cfg.max_iters - t)):
            be.iterate(t, limbs)
            _allreduce(dist, limbs, dist.ReduceOp.SUM, group)
            be.converge(t, limbs, eta)
            t += 1
        done, _ = be.status()
        if done:
            break
        chunk = min(chunk * 2, 32)
    # 4. global first-appearance numbering: MIN over ranks per component
    slots = words // (1 + 2 * d)
    minima = be.new(slots, "i64")
    be.components(offset, minima)
    _allreduce(dist, minima, dist.ReduceOp.MIN, group)
    if labels_out is None:
        labels_out = be.new(n_local, "i64")
    k, iters, mv, conv = be.finish(minima, labels_out, cfg.max_iters)
    if not return_result:
        return iters
    kk, fp = be.trace(iters)
    labels = labels_out.cpu().numpy() if hasattr(labels_out, "cpu") else np.asarray(labels_out)
    # a shard's labels need not cover [0, k): no Labeling validation here
    local = ShardLabels(labels=labels, k=k, modes=be.modes(k, d), offset=offset)
    return local, ShiftTrace(iterations=iters, total_movement_per_iter=mv, converged=conv,
                             cells_per_iter=kk, fingerprint_per_iter=fp)


class ShardLabels:
    """Labels of one rank's rows (global first-appearance numbering), the
    global cluster count and modes (identical on every rank)."""

    def __init__(self, labels, k, modes, offset):
        self.labels, self.k, self.modes, self.offset = labels, k, modes, offset

    def gather(self, parts) -> Labeling:
        """Concatenate all ranks' parts (in rank order) into a Labeling."""
        return Labeling(labels=np.concatenate([p.labels for p in parts]), k=self.k, modes=self.modes)
