"""Hypothesis properties on the CUDA engine, mirroring the reference's own
property tests (test_grid.py:72-89,134-145,190-205; test_modeseek.py:
369-382,555-562) -- with the exact-arithmetic model (tests/exact_model.py)
as a bitwise expectation where the reference only has a tolerance."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2104_00303_b200 as gs
from oracle import gridshift_oracle as O
from tests import exact_model as X

pytestmark = pytest.mark.gpu


@pytest.mark.usefixtures("exact_sums")
@settings(max_examples=40)
@given(st.integers(1, 4), st.integers(1, 60), st.sampled_from([0.25, 0.7, 1.0]), st.integers(0, 2**31 - 1))
def test_step_bitwise_exact_model(d, n, h, seed):
    # test_modeseek.py:369-382 (reference: rtol 1e-9 vs the linear-scan oracle)
    y = np.random.default_rng(seed).uniform(-4, 4, size=(n, d))
    moved, mv = gs.meanshiftpp_step(gs.PointSet(y), gs.ShiftConfig(h=h))
    P = X.Params(y, h)
    want, wmv, _, _ = X.shift_once(y, h, P)
    assert np.array_equal(moved.data, want)
    assert mv == wmv
    # and the reference oracle within its own tolerance
    y2, mv2 = O.shift_once(y, h)
    assert np.allclose(moved.data, y2, rtol=1e-9, atol=1e-12)
    assert mv == pytest.approx(mv2, rel=1e-9, abs=1e-12)


@given(seed=st.integers(0, 10_000), n=st.integers(1, 200), d=st.integers(1, 4), h=st.floats(0.05, 3.0))
def test_mass_conservation(seed, n, d, h):
    # test_grid.py:134-145
    data = np.random.default_rng(seed).normal(0, 2, size=(n, d))
    t = gs.build_cell_tables(gs.PointSet(data), h)
    assert int(t.counts.sum()) == n
    assert np.all(t.counts >= 1)
    ref, _ = O.cell_tables(data, h)
    assert np.array_equal(t.cells, ref.cells) and np.array_equal(t.counts, ref.counts)


@given(seed=st.integers(0, 10_000), d=st.integers(1, 4))
def test_neighbourhood_bitwise_reference_order(seed, d):
    # reference-order sums (the default): tables and neighbourhood sums equal
    # the reference's (the oracle reproduces them bitwise, test_oracle.py)
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    data = rng.normal(0.0, 3.0, size=(n, d))
    h = float(rng.uniform(0.2, 2.0))
    t = gs.neighbor_stats(gs.PointSet(data), h)
    ref, _ = O.cell_tables(data, h)
    nc, ns = O.neighbour_stats(ref)
    assert np.array_equal(t.cells, ref.cells) and np.array_equal(t.counts, ref.counts)
    assert np.array_equal(t.sums, ref.sums)
    assert np.array_equal(t.nbr_counts, nc) and np.array_equal(t.nbr_sums, ns)


@pytest.mark.usefixtures("exact_sums")
@given(seed=st.integers(0, 10_000), d=st.integers(1, 3))
def test_neighbourhood_equals_linear_scan(seed, d):
    # test_grid.py:190-205: counts bitwise, sums = exactly rounded scan sums
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 80))
    data = rng.uniform(1.0, 6.0, size=(n, d))
    h = float(rng.uniform(0.2, 2.0))
    t = gs.neighbor_stats(gs.PointSet(data), h)
    cells = np.floor(data / h).astype(np.int64)
    for r in range(t.k):
        mask = (np.abs(cells - t.cells[r]) <= 1).all(axis=1)
        assert int(t.nbr_counts[r]) == int(mask.sum())
        assert t.nbr_sums[r].tolist() == [math.fsum(data[mask, j]) for j in range(d)]


@settings(max_examples=30)
@given(st.integers(2, 40), st.integers(0, 2**31 - 1))
def test_extraction_partition(n, seed):
    # test_modeseek.py:555-562, plus equality with the oracle's labels
    y = np.random.default_rng(seed).uniform(-3, 3, size=(n, 2))
    lab = gs.extract_clusters(gs.PointSet(y), 0.5)
    assert set(np.unique(lab.labels)) == set(range(lab.k))
    labels, k, modes = O.extract(y, 0.5)
    assert np.array_equal(lab.labels, labels) and lab.k == k
    assert np.allclose(lab.modes, modes, rtol=0, atol=1e-12)


@pytest.mark.usefixtures("exact_sums")
@settings(max_examples=25)
@given(st.integers(1, 3), st.integers(5, 400), st.sampled_from([0.3, 0.6, 1.1]), st.integers(0, 2**31 - 1))
def test_full_run_bitwise_exact_model(d, n, h, seed):
    y = np.random.default_rng(seed).normal(0, 1.5, size=(n, d))
    lab, tr = gs.meanshiftpp(gs.PointSet(y), gs.ShiftConfig(h=h))
    m = X.meanshiftpp(y, h)
    assert tr.iterations == m["iterations"]
    np.testing.assert_array_equal(tr.total_movement_per_iter, m["movement"])
    assert np.array_equal(lab.labels, m["labels"]) and np.array_equal(lab.modes, m["modes"])
    r = O.meanshiftpp(y, h)
    assert np.array_equal(lab.labels, r["labels"])


@given(st.sampled_from([0.5, 1.0, 2.0]), st.lists(st.floats(-1e6, 1e6), min_size=1, max_size=4),
       st.lists(st.integers(-1000, 1000), min_size=1, max_size=4))
def test_bin_translation_covariance(h, point, k):
    # test_grid.py:72-89 through the device tables: cells shift by k
    d = min(len(point), len(k))
    point, k = np.array(point[:d]), np.array(k[:d])
    q = point / h
    sq = (point + h * k) / h
    if np.min(np.abs(q - np.round(q))) <= 1e-6 or np.min(np.abs(sq - np.round(sq))) <= 1e-6:
        return
    a = gs.build_cell_tables(gs.PointSet(point[None, :]), h).cells[0]
    b = gs.build_cell_tables(gs.PointSet((point + h * k)[None, :]), h).cells[0]
    assert np.array_equal(b, a + k)


def test_invalid_inputs():
    for bad in (np.array([[np.nan, 1.0]]), np.array([[np.inf]]), np.empty((0, 2)), np.array([1.0, 2.0])):
        with pytest.raises(ValueError):
            gs.meanshiftpp(gs.PointSet(bad), gs.ShiftConfig(1.0))
    with pytest.raises(ValueError):
        gs.ShiftConfig(h=-1.0)
    with pytest.raises(ValueError):
        gs.ShiftConfig(h=1.0, max_iters=0)
    with pytest.raises(ValueError):
        gs.meanshiftpp(gs.PointSet(np.zeros((3, 9))), gs.ShiftConfig(1.0))   # d > 8: engine envelope


@pytest.mark.usefixtures("exact_sums")
@settings(max_examples=20)
@given(st.integers(4, 8), st.integers(5, 300), st.sampled_from([0.6, 1.0, 1.7]), st.booleans(),
       st.integers(0, 2**31 - 1))
def test_full_run_high_d_bitwise_exact_model(d, n, h, spread, seed):
    # d = 4..8: dense or hash tables (a wide spread forces the hash path),
    # k_agg_warp / k_agg, register-prefetched k_shift
    rng = np.random.default_rng(seed)
    y = rng.normal(0, 40.0 if spread else 1.2, size=(n, d))
    lab, tr = gs.meanshiftpp(gs.PointSet(y), gs.ShiftConfig(h=h, max_iters=40))
    m = X.meanshiftpp(y, h, None, 40)
    assert tr.iterations == m["iterations"]
    np.testing.assert_array_equal(tr.total_movement_per_iter, m["movement"])
    assert np.array_equal(lab.labels, m["labels"]) and np.array_equal(lab.modes, m["modes"])


@pytest.mark.usefixtures("exact_sums")
def test_large_hash_run_equals_exact_model():
    # a sorted (n >= 32768) run on a hash table (d = 4, wide box)
    rng = np.random.default_rng(77)
    centers = rng.uniform(-300, 300, size=(12, 4))
    y = (centers[rng.integers(0, 12, size=60_000)] + rng.normal(0, 1.5, size=(60_000, 4)))
    lab, tr = gs.meanshiftpp(gs.PointSet(y), gs.ShiftConfig(h=1.0, eta=1e-3, max_iters=30))
    m = X.meanshiftpp(y, 1.0, 1e-3, 30)
    assert tr.iterations == m["iterations"]
    np.testing.assert_array_equal(tr.total_movement_per_iter, m["movement"])
    assert np.array_equal(lab.labels, m["labels"]) and np.array_equal(lab.modes, m["modes"])
