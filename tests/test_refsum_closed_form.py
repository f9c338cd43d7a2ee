"""The closed form behind the reference-order sums (gs_refsum.cuh
seqsum_mag_from), compiled for the host from the same header, against
sequential numpy addition -- np.add.accumulate adds left to right exactly
as np.bincount accumulates a cell's points (grid.py:186-187)."""

import os
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
SRC = HERE / "native" / "seqsum_check.cu"


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path_factory.mktemp("seqsum") / "seqsum_check"
    subprocess.run([nvcc, "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", str(exe), str(SRC)], check=True,
                   capture_output=True, timeout=600)
    return exe


def _cases(seed=0, count=3000):
    rng = np.random.default_rng(seed)
    out = []
    for t in range(count):
        c = int(rng.integers(1, 3000))
        a = float(abs(rng.normal(0, 10.0 ** rng.uniform(-3, 3))))
        if t % 4 == 0:               # few mantissa bits: ties
            a = float(np.round(a * 64) / 64)
        if t % 7 == 0:               # integers (image features)
            a = float(rng.integers(0, 256))
        s0 = 0.0
        if t % 3 == 1:               # continue from a running sum
            s0 = float(abs(rng.normal(0, 10.0 ** rng.uniform(-2, 5))))
        if t % 11 == 0:              # a exactly half an ulp of s0
            s0 = float(2.0 ** int(rng.integers(-5, 20)) * (1 + int(rng.integers(0, 1000)) * 2.0 ** -52))
            a = float(np.spacing(s0) / 2)
        out.append((s0, a, c))
    return out


def _seq(s0, a, c):
    return float(np.add.accumulate(np.r_[s0, np.full(c, a)])[-1])


def test_closed_form_equals_sequential_addition(harness):
    cases = _cases()
    inp = "".join(f"{np.float64(s).view(np.uint64):x} {np.float64(a).view(np.uint64):x} {c}\n"
                  for s, a, c in cases)
    r = subprocess.run([str(harness)], input=inp, capture_output=True, text=True, check=True, timeout=120)
    got = [int(x, 16) for x in r.stdout.split()]
    assert len(got) == len(cases)
    bad = []
    for (s, a, c), g in zip(cases, got):
        want = int(np.float64(_seq(s, a, c)).view(np.uint64))
        if g != want:
            bad.append((s, a, c, hex(g), hex(want)))
    assert not bad, bad[:5]
