"""The C ABI library builds for sm_100a, loads without a GPU, and exports
exactly the entry points include/gridshift_cuda.h declares."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2104_00303_b200 import _build, _lib

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "gridshift_cuda.h"


def declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"GS_API\s+[\w\s\*]+?\b(gs_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def test_header_declares_entry_points():
    names = declared()
    assert "gs_meanshiftpp" in names and "gs_track_sequence" in names
    assert names == sorted(_lib.SIGNATURES), "ctypes table must mirror the header"


def declared_arity():
    txt = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    out = {}
    for m in re.finditer(r"GS_API\s+[\w\s\*]+?\b(gs_\w+)\s*\(([^)]*)\)", txt):
        args = [a for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        out[m.group(1)] = len(args)
    return out


def test_ctypes_arity_matches_header():
    ar = declared_arity()
    for name, (_, args) in _lib.SIGNATURES.items():
        assert len(args) == ar[name], name


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(gs_\w+)", out))
    assert exported == set(declared())
    for name in declared():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_version_and_error_strings(lib):
    assert b"sm_100a" in lib.gs_version()
    assert lib.gs_last_error() == b""


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_context_is_rejected(lib):
    rc = lib.gs_meanshiftpp(None, None, 1, 1, 1.0, 1.0, 1, None, None, None, None, None)
    assert rc == _lib.GS_EINVAL


def _build_c_host(tmp_path):
    exe = tmp_path / "c_host"
    libdir = ROOT / "paper_2104_00303_b200"
    subprocess.run(["gcc", "-O2", "-I", str(ROOT / "include"), str(ROOT / "examples" / "c_host.c"),
                    "-L", str(libdir), "-lgridshift_cuda", f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)],
                   check=True)
    return exe


def test_c_host_links_against_the_header_and_library(lib, tmp_path):
    # a plain C caller (no Python): compiles against include/gridshift_cuda.h,
    # links libgridshift_cuda.so and loads it (no GPU needed for --version)
    exe = _build_c_host(tmp_path)
    out = subprocess.run([str(exe), "--version"], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


@pytest.mark.gpu
def test_c_host_runs_the_engine(lib, tmp_path):
    exe = _build_c_host(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert "k=2 " in out and "converged=1" in out
    modes = sorted(tuple(float(v) for v in line.split("(")[1].rstrip(")").split(","))
                   for line in out.splitlines() if line.startswith("mode "))
    assert abs(modes[0][0] - 2.0) < 0.05 and abs(modes[1][0] - 8.0) < 0.05
