"""ctypes binding of `libgridshift_cuda.so` (C ABI: include/gridshift_cuda.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every engine call raises.  Status codes map to the reference's
error convention: GS_EINVAL / GS_EUNSUPPORTED -> ValueError,
GS_ERUNTIME -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("GRIDSHIFT_LIB", Path(__file__).resolve().parent / "libgridshift_cuda.so"))

GS_OK, GS_EINVAL, GS_ERUNTIME, GS_EUNSUPPORTED = 0, 1, 2, 3
GS_DTYPE_F64, GS_DTYPE_F32 = 0, 1
GS_OPT_COLLAPSED = 1
GS_OPT_SUMS, GS_SUMS_REFERENCE, GS_SUMS_EXACT, GS_SUMS_SEQMODEL = 2, 0, 1, 2

_P = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_f64 = C.c_double

# symbol -> (restype, argtypes); mirrors include/gridshift_cuda.h
SIGNATURES = {
    "gs_last_error": (C.c_char_p, []),
    "gs_version": (C.c_char_p, []),
    "gs_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "gs_ctx_destroy": (None, [_P]),
    "gs_meanshiftpp": (C.c_int, [_P, _P, _i64, _i32, _f64, _f64, _i32, _P, _P, _P, _P, _P]),
    "gs_meanshiftpp_host": (C.c_int, [_P, _P, _i32, _i64, _i32, _f64, _f64, _i32, _P, _P, _P, _P, _P]),
    "gs_meanshiftpp_device": (C.c_int, [_P, _P, _i32, _i64, _i32, _f64, _f64, _i32, _P, _P, _P,
                                        _P, _P, _P]),
    "gs_segment_image": (C.c_int, [_P, _P, _i32, _i32, _i32, _f64, _f64, _f64, _i32, _P, _P, _P,
                                   _P, _P]),
    "gs_fetch_modes": (C.c_int, [_P, _P, _i64]),
    "gs_fetch_mean_colors": (C.c_int, [_P, _P, _i64]),
    "gs_ctx_set_option": (C.c_int, [_P, _i32, _i64]),
    "gs_fetch_trace": (C.c_int, [_P, _P, _P, _i32]),
    "gs_fetch_shift_bytes": (C.c_int, [_P, _P, _i32]),
    "gs_fetch_iterate": (C.c_int, [_P, _P, _i64]),
    "gs_fetch_refsum_stats": (C.c_int, [_P, _P, _i32]),
    "gs_fetch_transfer_bytes": (C.c_int, [_P, _P, _P]),
    "gs_profile": (C.c_int, [_P, _i32, _P, _P, _i32]),
    "gs_profile_kind": (C.c_char_p, [_i32]),
    "gs_shift_step": (C.c_int, [_P, _P, _i64, _i32, _f64, _P, _P]),
    "gs_build_tables": (C.c_int, [_P, _P, _i64, _i32, _f64, _i64, _P, _P, _P, _P, _P, _P]),
    "gs_extract_clusters": (C.c_int, [_P, _P, _i64, _i32, _f64, _P, _P]),
    "gs_track_sequence": (C.c_int, [_P, _P, _i32, _i32, _i32, _f64, _f64, _i32, _i32, _P, _i32,
                                    _f64, _i32, _i32, _f64, _i32, _P, _P, _P, _P, _P, _P]),
    "gs_fetch_track_bins": (C.c_int, [_P, _P, _i32, _P]),
    "gs_shard_init": (C.c_int, [_P, _P, _i32, _i64, _i32, _f64, _P, _P, _P, _P, _P]),
    "gs_shard_plan": (C.c_int, [_P, _P, _P, _P, _i32, _i64, _i32, _P, _P]),
    "gs_shard_table_io": (C.c_int, [_P, _P, _i32, _P]),
    "gs_shard_iterate": (C.c_int, [_P, _i32, _P, _P]),
    "gs_shard_converge": (C.c_int, [_P, _i32, _P, _f64, _P]),
    "gs_shard_status": (C.c_int, [_P, _P, _P, _P]),
    "gs_shard_components": (C.c_int, [_P, _i64, _P, _P, _P]),
    "gs_shard_finish": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
}

_lib = None
_lock = threading.Lock()
_tls = threading.local()


def load():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH.name} is not built; run `python -c \"import __graft_entry__ as g; "
                    f"g.build()\"` (nvcc, sm_100a). There is no CPU fallback.")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == GS_OK:
        return
    msg = (load().gs_last_error() or b"").decode(errors="replace")
    if rc in (GS_EINVAL, GS_EUNSUPPORTED):
        raise ValueError(msg)
    raise RuntimeError(msg or f"gridshift CUDA error {rc}")


def default_device() -> int:
    return int(os.environ.get("GRIDSHIFT_DEVICE", os.environ.get("LOCAL_RANK", "0")))


class _Contexts(dict):
    """This thread's engine contexts (device -> gs_ctx*).  Held in a
    threading.local, so it is released when its thread exits: every context
    (streams, events, pinned and device buffers) is destroyed then, and a
    long-lived process whose callers come from short-lived worker threads
    (cli.py:206-216 opens a ThreadPoolExecutor per call) does not leak."""

    def __del__(self):
        lib = _lib
        if lib is None:
            return
        for ctx in self.values():
            try:
                lib.gs_ctx_destroy(ctx)
            except Exception:   # noqa: BLE001 -- interpreter shutdown
                pass
        self.clear()


def context(device: int | None = None) -> C.c_void_p:
    """Per-thread, per-device engine context (contexts serialise calls, so
    concurrent callers each get their own, cli.py:206-216 style); destroyed
    when the thread exits (_Contexts)."""
    dev = default_device() if device is None else int(device)
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = _Contexts()
    ctx = cache.get(dev)
    if ctx is None:
        out = _P()
        check(load().gs_ctx_create(dev, C.byref(out)))
        ctx = cache[dev] = out
    return ctx


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(_P)


def ref(x):
    return C.byref(x)


N_KINDS = 13


def profile(mode: int, device: int | None = None):
    """Kernel accounting of this thread's context (see gs_profile)."""
    ms = np.zeros(N_KINDS)
    cnt = np.zeros(N_KINDS, dtype=np.int64)
    check(load().gs_profile(context(device), mode, ptr(ms), ptr(cnt), N_KINDS))
    if mode != 2:
        return None
    names = [load().gs_profile_kind(i).decode() for i in range(N_KINDS)]
    return {nm: (float(ms[i]), int(cnt[i])) for i, nm in enumerate(names)}
