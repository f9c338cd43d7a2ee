"""Build the in-tree CUDA library `libgridshift_cuda.so` (sm_100a) with nvcc.

The .so is git-ignored but travels to the GPU box with the repo snapshot;
cudart is linked statically so the library does not depend on the CUDA
runtime bundled with torch.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libgridshift_cuda.so"
SOURCES = ["gs_engine.cu"]
HEADERS = ["gs_common.cuh", "gs_kernels.cuh", "gs_refsum.cuh", "gs_track.cuh"]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
]
# development only: e.g. GS_NVCC_EXTRA="-DGS_ONLY_D=3" builds one dimension (8x faster)
NVCC_FLAGS += os.environ.get("GS_NVCC_EXTRA", "").split()


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libgridshift_cuda.so")


STAMP = LIB.with_name(LIB.name + ".srchash")


def source_hash() -> str:
    """Content hash of everything the library is built from (mtimes do not
    survive the snapshot to the GPU box; content does)."""
    import hashlib

    hsh = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for p in [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "gridshift_cuda.h"]:
        hsh.update(p.name.encode())
        hsh.update(p.read_bytes())
    return hsh.hexdigest()


def stale() -> bool:
    if not LIB.exists() or not STAMP.exists():
        return True
    return STAMP.read_text().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, "-shared", "-o", str(tmp),
           *[str(CSRC / s) for s in SOURCES], "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    tmp.replace(LIB)
    STAMP.write_text(source_hash() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
