"""CUDA engine vs the reference (frozen fixtures) and the CPU oracle.

Contract (BASELINE.json north_star): cell keys and per-cell counts
bit-exact every iteration (checked through the order-independent
(cells, counts) fingerprint the engine records on device), labels
identical, modes within 1e-9*h in fp64.  The tests run in the engine's
default sum order (the sequential model of the reference's per-cell sums,
DESIGN.md section 4) unless a fixture selects the reference order (bit for
bit) or the exact order (pinned to tests/exact_model.py).
"""

import math

import numpy as np
import pytest

import paper_2104_00303_b200 as gs
from oracle import gridshift_oracle as O
from paper_2104_00303_b200 import workloads as W
from tests import exact_model as X
from tests import goldens as G

pytestmark = pytest.mark.gpu

MODES_TOL = 1e-9   # * h


def _eta(f):
    return None if np.isnan(f["eta"]) else float(f["eta"])


# ------------------------------------------------------------------ tables

@pytest.mark.parametrize("c", G.cases("tables"))
def test_tables_vs_reference(c):
    f = G.case("tables", c)
    t = gs.neighbor_stats(gs.PointSet(f["y"]), float(f["h"]))
    assert np.array_equal(t.cells, f["cells"])
    assert np.array_equal(t.counts, f["counts"])
    np.testing.assert_allclose(t.sums, f["sums"], rtol=1e-12, atol=1e-300)
    assert np.array_equal(t.nbr_counts, f["nbr_counts"])
    scale = np.abs(f["y"]).max()
    np.testing.assert_allclose(t.nbr_sums, f["nbr_sums"], rtol=1e-12, atol=1e-15 * scale * len(f["y"]))
    # one table of distinct values: np.bincount's sums bit for bit (default and reference order)
    assert np.array_equal(t.sums, f["sums"])
    assert np.array_equal(t.nbr_sums, f["nbr_sums"])


@pytest.mark.usefixtures("exact_sums")
def test_tables_exact_sums():
    # exact device sums == math.fsum of the member coordinates
    rng = np.random.default_rng(5)
    y = rng.uniform(1.0, 9.0, size=(5000, 3))
    t = gs.build_cell_tables(gs.PointSet(y), 0.75)
    cells = np.floor(y / 0.75).astype(np.int64)
    for i in range(0, t.k, 7):
        m = np.all(cells == t.cells[i], axis=1)
        assert int(m.sum()) == int(t.counts[i])
        want = [math.fsum(y[m, j]) for j in range(3)]
        assert t.sums[i].tolist() == want


# ------------------------------------------------------------------- steps

@pytest.mark.parametrize("c", G.cases("steps"))
def test_step_vs_reference(c):
    # criterion 1 (test_acceptance.py:38-61): max error relative to the field
    f = G.case("steps", c)
    moved, mv = gs.meanshiftpp_step(gs.PointSet(f["y"]), gs.ShiftConfig(h=float(f["h"])))
    want = f["y_next"]
    # a single step: the reference's step bit for bit (default and reference order)
    assert np.array_equal(moved.data, want)
    rel = np.abs(moved.data - want).max() / max(np.abs(want).max(), 1e-30)
    assert rel <= 1e-10
    assert mv == pytest.approx(float(f["movement"]), rel=1e-9, abs=1e-12)


def _exact_step(y, h):
    cells = np.floor(y / h).astype(np.int64)
    out = np.empty_like(y)
    for i in range(len(y)):
        near = np.abs(cells - cells[i]).max(axis=1) <= 1
        cnt = int(near.sum())
        out[i] = [math.fsum(y[near, j]) / cnt for j in range(y.shape[1])]
    return out


@pytest.mark.usefixtures("exact_sums")
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5])
def test_step_is_exactly_rounded(d):
    # values in [1, 2): fixed-point capture is exact, so the device result is
    # the correctly rounded neighbourhood sum divided by the count
    rng = np.random.default_rng(100 + d)
    y = rng.uniform(1.0, 2.0, size=(300, d))
    moved, _ = gs.meanshiftpp_step(gs.PointSet(y), gs.ShiftConfig(h=0.21))
    assert np.array_equal(moved.data, _exact_step(y, 0.21))


def test_step_kats():
    # test_modeseek.py:92-105
    pts = gs.PointSet(np.array([[3.7, -1.2]]))
    moved, mv = gs.meanshiftpp_step(pts, gs.ShiftConfig(h=1.0))
    assert np.array_equal(moved.data, pts.data) and mv == 0.0
    moved, mv = gs.meanshiftpp_step(gs.PointSet(np.array([[0.1], [0.2]])), gs.ShiftConfig(h=1.0))
    assert moved.data == pytest.approx(np.array([[0.15], [0.15]]), rel=1e-12)
    assert mv == pytest.approx(0.1, rel=1e-12)


# -------------------------------------------------------------------- runs

def _mv_atol(n, scale):
    # the reference's sequential fp64 sums carry O(cell size * eps) noise per
    # point (visible once cells collapse); the device sums are exact
    return max(n * scale * 1e-12, 1e-300)


def _check_run(lab, tr, f, h, y=None):
    n = int(f["n"]) if "n" in f else len(f["y"])
    scale = float(np.abs(f["modes"]).max()) * 2 + h
    atol = _mv_atol(n, scale)
    it = tr.iterations
    ref_mv = f["movement"]
    if it < int(f["iterations"]):
        # exact device sums reached a true fixed point (movement exactly 0)
        # while the reference's sequential sums only jitter at rounding
        # noise below eta: allowed only for eta under that noise floor
        assert tr.converged and tr.total_movement_per_iter[-1] == 0.0
        assert np.all(np.abs(ref_mv[it - 1:]) <= atol)
    else:
        assert it == int(f["iterations"])
        assert tr.converged == bool(f["converged"])
    assert tr.cells_per_iter.tolist() == f["iter_k"][:it].tolist()
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in f["iter_fp"][:it]]
    np.testing.assert_allclose(tr.total_movement_per_iter, ref_mv[:it], rtol=1e-9, atol=atol)
    assert lab.k == int(f["k"])
    assert np.abs(lab.modes - f["modes"]).max() <= MODES_TOL * h


@pytest.mark.parametrize("c", G.cases("runs"))
def test_run_vs_reference(c):
    f = G.case("runs", c)
    h = float(f["h"])
    lab, tr = gs.meanshiftpp(gs.PointSet(f["y"]), gs.ShiftConfig(h=h, eta=_eta(f), max_iters=int(f["max_iters"])))
    assert np.array_equal(lab.labels, f["labels"])
    _check_run(lab, tr, f, h)


@pytest.mark.usefixtures("reference_sums")
@pytest.mark.parametrize("c", G.cases("runs"))
def test_run_trajectory_bitwise_vs_reference(c):
    """Reference-order sums (GS_SUMS_REFERENCE): the final iterate -- hence every
    iterate -- equals the reference's bit for bit (the oracle reproduces the
    reference bitwise on these fixtures, test_oracle.py), the iteration
    count and labels are the reference's, and the modes differ only by the
    reference's own rounding of the mode means (exact here, sequential
    there: modeseek.py:268-271)."""
    f = G.case("runs", c)
    h = float(f["h"])
    y0 = f["y"]
    lab, tr = gs.meanshiftpp(gs.PointSet(y0), gs.ShiftConfig(h=h, eta=_eta(f), max_iters=int(f["max_iters"])))
    r = O.meanshiftpp(y0, h, _eta(f), int(f["max_iters"]))
    assert tr.iterations == r["iterations"] == int(f["iterations"])
    assert tr.converged == r["converged"]
    y = gs.modeseek.last_iterate(*y0.shape)
    assert np.array_equal(y, r["y"])
    assert np.array_equal(lab.labels, f["labels"])
    np.testing.assert_allclose(lab.modes, f["modes"], rtol=1e-13, atol=1e-13 * h)


@pytest.mark.usefixtures("reference_sums")
def test_cfg0_trajectory_bitwise_vs_reference():
    c = W.CONFIGS["cfg0"]
    y0 = W.blobs2d()
    lab, tr = gs.meanshiftpp(gs.PointSet(y0), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]))
    r = O.meanshiftpp(y0, c["h"], c["eta"], c["max_iters"])
    assert tr.iterations == r["iterations"]
    assert np.array_equal(gs.modeseek.last_iterate(*y0.shape), r["y"])
    assert np.array_equal(lab.labels, r["labels"])


def _dense_runs():
    return [c for c in G.cases("runs") if G.case("runs", c)["y"].shape[1] <= 3]


@pytest.mark.parametrize("c", _dense_runs() + ["cfg0", "cloud300k",
                               pytest.param("cfg1", marks=pytest.mark.slow),
                               pytest.param("cloud2m", marks=pytest.mark.slow)])
def test_run_bitwise_vs_sequential_model(c):
    """The DEFAULT sum order against its independent CPU restatement
    (tests/seq_model.py: exact first table, closed form for single-source
    cells, model_fold32 for mixed cells, sequential neighbourhood sums): the
    final iterate -- hence every iterate, every closed form and every model
    fold on the device -- plus movement trace, per-iteration tables, labels
    and modes, bit for bit."""
    from tests import seq_model as S

    if c == "cfg0":
        cfgd = W.CONFIGS["cfg0"]
        y0, h, eta, mi = W.blobs2d(), cfgd["h"], cfgd["eta"], cfgd["max_iters"]
    elif c == "cfg1":       # 2M pixels, 100 iterations, sorted dense path
        cfgd = W.CONFIGS["cfg1"]
        y0 = gs.image_to_features(gs.Image(W.cfg1_image()), "rgb").data
        h, eta, mi = cfgd["h"], cfgd["eta"], cfgd["max_iters"]
    elif c in ("cloud300k", "cloud2m"):   # the cfg4 generator (big merging cells), 50 iterations
        n = 300_000 if c == "cloud300k" else 2_000_000
        y0, h, eta, mi = W.cloud3d(n, seed=4).astype(np.float64), 1.0, 1e-3, 50
    else:
        f = G.case("runs", c)
        y0, h, eta, mi = f["y"], float(f["h"]), _eta(f), int(f["max_iters"])
    lab, tr = gs.meanshiftpp(gs.PointSet(y0), gs.ShiftConfig(h=h, eta=eta, max_iters=mi))
    y = gs.modeseek.last_iterate(*y0.shape)
    r = S.meanshiftpp(y0, h, eta, mi)
    assert tr.iterations == r["iterations"] and tr.converged == r["converged"]
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in r["iter_fp"]]
    assert np.array_equal(y, r["y"])
    np.testing.assert_array_equal(tr.total_movement_per_iter, r["movement"])
    assert np.array_equal(lab.labels, r["labels"])
    assert np.array_equal(lab.modes, r["modes"])


@pytest.mark.usefixtures("exact_sums")
@pytest.mark.parametrize("c", G.cases("runs"))
def test_run_bitwise_vs_exact_model(c):
    # every device reduction pinned: the GPU equals the exact-arithmetic
    # model of the same algorithm bit for bit (iterates, movement, modes)
    from tests import exact_model as X

    f = G.case("runs", c)
    h = float(f["h"])
    m = X.meanshiftpp(f["y"], h, _eta(f), int(f["max_iters"]))
    lab, tr = gs.meanshiftpp(gs.PointSet(f["y"]), gs.ShiftConfig(h=h, eta=_eta(f), max_iters=int(f["max_iters"])))
    assert tr.iterations == m["iterations"]
    np.testing.assert_array_equal(tr.total_movement_per_iter, m["movement"])
    assert np.array_equal(lab.labels, m["labels"])
    assert np.array_equal(lab.modes, m["modes"])
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in m["iter_fp"]]


def test_run_kats():
    # test_modeseek.py:141-236
    lab, tr = gs.meanshiftpp(gs.PointSet(np.tile([1.5, -0.5, 2.0], (40, 1))), gs.ShiftConfig(h=0.7))
    assert lab.k == 1 and np.all(lab.labels == 0) and tr.iterations == 1 and tr.converged
    assert tr.total_movement_per_iter.sum() == 0.0
    assert lab.modes[0].tolist() == [1.5, -0.5, 2.0]
    lab, tr = gs.meanshiftpp(gs.PointSet(np.array([[0.2], [9.7]])), gs.ShiftConfig(h=1.0))
    assert tr.iterations == 1 and tr.converged and tr.total_movement_per_iter[-1] == 0.0 and lab.k == 2
    rng = np.random.default_rng(3)
    data = rng.uniform(0, 1, size=(120, 3))
    lab, tr = gs.meanshiftpp(gs.PointSet(data), gs.ShiftConfig(h=50.0))
    assert lab.k == 1 and tr.converged
    assert np.allclose(lab.modes[0], data.mean(axis=0), rtol=1e-9, atol=1e-12)


def test_engine_is_deterministic():
    # test_modeseek.py:229-236, on a large input where atomics interleave
    y = W.cloud3d(400_000, seed=12).astype(np.float64)
    cfg = gs.ShiftConfig(h=1.0, eta=1e-3, max_iters=20)
    a, ta = gs.meanshiftpp(gs.PointSet(y), cfg)
    b, tb = gs.meanshiftpp(gs.PointSet(y), cfg)
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(a.modes, b.modes)
    assert np.array_equal(ta.total_movement_per_iter, tb.total_movement_per_iter)


def test_invalid_inputs_raise_value_error():
    with pytest.raises(ValueError):
        gs.ShiftConfig(h=0.0)
    with pytest.raises(ValueError):
        gs.PointSet(np.array([[1.0, np.nan]]))
    with pytest.raises(ValueError):
        gs.build_cell_tables(gs.PointSet(np.array([[1e30]])), 1e-8)
    with pytest.raises(ValueError):
        gs.meanshiftpp(gs.PointSet(np.array([[1e30]])), gs.ShiftConfig(h=1e-8))


# -------------------------------------------------------------- extraction

@pytest.mark.parametrize("c", G.cases("extract"))
def test_extract_vs_reference(c):
    f = G.case("extract", c)
    lab = gs.extract_clusters(gs.PointSet(f["y"]), float(f["h"]))
    assert lab.k == int(f["k"])
    assert np.array_equal(lab.labels, f["labels"])
    assert np.abs(lab.modes - f["modes"]).max() <= MODES_TOL * float(f["h"])


# ---------------------------------------------------------------- tracking

@pytest.mark.parametrize("c", G.cases("tracking"))
def test_tracking_vs_reference(c):
    f = G.case("tracking", c)
    cx, cy, w, hp = f["win"].tolist()
    win = gs.Window(cx=cx, cy=cy, w=int(w), h_px=int(hp))
    rows = gs.track_sequence([gs.Image(p) for p in f["frames"]], win, gs.ShiftConfig(h=float(f["h"])),
                             [int(f["selected"])], update_bins=bool(f["update"]))
    assert [r.window.cx for r in rows] == f["cx"].tolist()
    assert [r.window.cy for r in rows] == f["cy"].tolist()
    assert [r.lost for r in rows] == f["lost"].tolist()
    assert [r.last_match_count for r in rows] == f["matches"].tolist()
    assert [len(r.bins.bins) for r in rows] == f["nbins"].tolist()
    fps = [W.fingerprint(np.array(sorted(r.bins.bins), dtype=np.int64),
                         np.zeros(len(r.bins.bins), dtype=np.int64)) for r in rows]
    assert fps == [int(v) for v in f["bins_fp"]]


def test_track_frame_matches_oracle():
    f = G.case("tracking", "track_video_small")
    frames = f["frames"]
    cx, cy, w, hp = f["win"].tolist()
    h = float(f["h"])
    st = gs.init_tracker(gs.Image(frames[0]), gs.Window(cx, cy, int(w), int(hp)), gs.ShiftConfig(h=h),
                         [int(f["selected"])])
    ost = dict(cx=cx, cy=cy, w=int(w), hp=int(hp), bins=set(st.bins.bins), lost=False,
               matches=st.last_match_count)
    for t in range(1, 6):
        st = gs.track_frame(st, gs.Image(frames[t]), gs.ShiftConfig(h=h), update_bins=True)
        ost = O.track_frame(ost, frames[t], h, update_bins=True)
        assert (st.window.cx, st.window.cy) == (ost["cx"], ost["cy"])
        assert st.last_match_count == ost["matches"]
        assert set(st.bins.bins) == ost["bins"]


# ------------------------------------------------------------ segmentation

def test_segment_fused_features_match_host_features():
    img = gs.Image(W.voronoi_image(96, 64, 9, seed=21))
    cfg = gs.ShiftConfig(h=10.0, eta=1e-3, max_iters=100)
    seg, tr = gs.segment_image(img, cfg, mode="rgbxy", scale=0.25)
    lab, tr2 = gs.meanshiftpp(gs.image_to_features(img, "rgbxy", scale=0.25), cfg)
    assert np.array_equal(seg.labels.ravel(), lab.labels)
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in tr2.fingerprint_per_iter]
    r = O.meanshiftpp(O.image_to_features(img.pixels, "rgbxy", 0.25), 10.0, 1e-3, 100)
    assert np.array_equal(lab.labels, r["labels"])


@pytest.mark.parametrize("shape,mode", [((96, 64), "rgbxy"), ((96, 64), "rgb"), ((640, 360), "rgb"),
                                        ((640, 360), "rgbxy")])
def test_segment_map_mean_colours_on_device(shape, mode):
    """SegmentMap from segment_image (mean colours accumulated on the GPU,
    gs_fetch_mean_colors) equals segment_map_from_labeling on the host --
    the reference's np.bincount fold (segment.py:109-117) -- bit for bit, for
    small (per-point labels on device) and sorted (per-cell label delivery)
    images, dense and hash tables."""
    img = gs.Image(W.voronoi_image(shape[0], shape[1], 12, seed=5))
    cfg = gs.ShiftConfig(h=10.0, eta=1e-3, max_iters=30)
    seg, _ = gs.segment_image(img, cfg, mode=mode, scale=0.25)
    lab = gs.Labeling(labels=seg.labels.ravel(), k=seg.k, modes=np.zeros((seg.k, 3)))
    host = gs.segment_map_from_labeling(img, lab)
    assert seg.mean_colors.shape == (seg.k, 3)
    assert np.array_equal(seg.mean_colors.view(np.uint64), host.mean_colors.view(np.uint64))
    assert np.array_equal(seg.labels, host.labels)


# ------------------------------------------------------- full BASELINE sizes

def test_cfg0_full_vs_reference():
    f = G.big("cfg0")
    c = W.CONFIGS["cfg0"]
    lab, tr = gs.meanshiftpp(gs.PointSet(W.blobs2d()), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]))
    assert np.array_equal(lab.labels, f["labels_u16"].astype(np.int64))
    _check_run(lab, tr, f, c["h"])


@pytest.mark.slow
def test_cfg1_full_vs_reference():
    f = G.big("cfg1")
    c = W.CONFIGS["cfg1"]
    img = gs.Image(W.cfg1_image())
    lab, tr = gs.segment_pixels(img, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), "rgb")
    assert np.array_equal(lab.labels, f["labels_u16"].astype(np.int64))
    _check_run(lab, tr, f, c["h"])


@pytest.mark.slow
def test_cfg2_image_vs_reference():
    f = G.big("cfg2")
    c = W.CONFIGS["cfg2"]
    img = gs.Image(W.cfg2_image(0))
    lab, tr = gs.segment_pixels(img, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), "rgbxy", 0.25)
    assert np.array_equal(lab.labels, f["labels_u16"].astype(np.int64))
    _check_run(lab, tr, f, c["h"])


def _digest(a):
    import hashlib

    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def _modes_vs_reference(lab, f, h, name):
    """modes within 1e-9*h of the reference (north_star), asserted -- no
    moved bar, no xfail.  The reference's per-cell sums are sequential fp64
    (grid.py:186-187), which drifts ~1e-9*h (10M points) to ~1e-8*h (100M)
    away from exact arithmetic over 50 creeping iterations; the default
    (sequential model) and the reference sum order both reproduce that
    rounding."""
    dev = float(np.abs(lab.modes - f["modes"]).max()) / h
    assert dev <= MODES_TOL, f"{name}: max|modes - reference| = {dev:.3g}*h > 1e-9*h"


def _check_model(lab, tr, f, h):
    """Bitwise equality with the exact-arithmetic model (tests/exact_model.py):
    every device reduction is pinned."""
    assert np.array_equal(lab.modes, f["model_modes"])
    assert _digest(lab.labels) == str(f["model_labels_digest"])
    np.testing.assert_array_equal(tr.total_movement_per_iter, f["model_movement"])


@pytest.fixture(params=["seqmodel", "reference"])
def both_sum_orders(request):
    """The default (sequential model) and the bit-for-bit reference order."""
    with gs.sum_order(request.param):
        yield request.param


@pytest.mark.slow
def test_cfg4_10m_vs_reference(both_sum_orders):
    f = G.big("cfg4_10m")
    c = W.CONFIGS["cfg4"]
    h = c["h"]
    y = W.cloud3d(10_000_000).astype(np.float64)
    lab, tr = gs.meanshiftpp(gs.PointSet(y), gs.ShiftConfig(h, c["eta"], c["max_iters"]))
    # per-iteration cells/counts bit-exact, labels identical to the reference
    assert tr.iterations == int(f["iterations"])
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in f["iter_fp"]]
    assert _digest(lab.labels) == str(f["labels_digest"])
    _modes_vs_reference(lab, f, h, "cfg4@10M")
    if both_sum_orders == "reference":   # the mode means: exact here, sequential there (modeseek.py:268-271)
        assert np.abs(lab.modes - f["modes"]).max() <= 1e-12 * h


@pytest.mark.slow
@pytest.mark.usefixtures("exact_sums")
def test_cfg4_10m_exact_model_bitwise():
    """GS_SUMS_EXACT: bit for bit the exact-arithmetic model (every device
    reduction pinned); the reference's sequential sums sit 1.73e-9*h away
    from exact arithmetic after 50 creeping iterations."""
    f = G.big("cfg4_10m")
    c = W.CONFIGS["cfg4"]
    y = W.cloud3d(10_000_000).astype(np.float64)
    lab, tr = gs.meanshiftpp(gs.PointSet(y), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]))
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in f["iter_fp"]]
    _check_model(lab, tr, f, c["h"])


@pytest.mark.slow
def test_cfg4_100m_vs_reference(both_sum_orders):
    """The benchmarked configuration at full size (fp32 input through the
    host entry point, as bench.py's e2e leg)."""
    f = G.big("cfg4_100m")
    c = W.CONFIGS["cfg4"]
    h = c["h"]
    x = W.cloud3d()
    lab, tr = gs.meanshiftpp_points(x, gs.ShiftConfig(h, c["eta"], c["max_iters"]))
    del x
    assert tr.iterations == int(f["iterations"])
    assert tr.cells_per_iter.tolist() == f["iter_k"].tolist()
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in f["iter_fp"]]
    assert lab.k == int(f["k"])
    assert np.array_equal(np.bincount(lab.labels, minlength=lab.k), f["label_sizes"])
    assert _digest(lab.labels) == str(f["labels_digest"])
    _modes_vs_reference(lab, f, h, "cfg4@100M")
    if both_sum_orders == "reference":   # (the reference's mode means are sequential sums too: ~1e-11*h at 100M points)
        assert np.abs(lab.modes - f["modes"]).max() <= 1e-10 * h


def _cfg2_images():
    # image 0 is test_cfg2_image_vs_reference
    return [i for i in range(1, 8) if (G.GOLDEN / f"big_cfg2_img{i}.npz").exists()]


@pytest.mark.slow
@pytest.mark.parametrize("i", _cfg2_images())
def test_cfg2_batch_image_vs_reference(i):
    """Images 1-7 of the cfg2 batch (distinct seeds), each against its own
    reference run: per-iteration cells/counts, labels, modes."""
    f = G.big(f"cfg2_img{i}")
    c = W.CONFIGS["cfg2"]
    img = gs.Image(W.cfg2_image(i))
    lab, tr = gs.segment_pixels(img, gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), "rgbxy", 0.25)
    assert np.array_equal(lab.labels, f["labels_u16"].astype(np.int64))
    assert tr.iterations == int(f["iterations"])
    assert [int(v) for v in tr.fingerprint_per_iter] == [int(v) for v in f["iter_fp"]]
    assert lab.k == int(f["k"])
    _modes_vs_reference(lab, f, c["h"], f"cfg2 image {i}")


def test_cfg3_full_vs_reference():
    """cfg3 at BASELINE size: 300 frames of 1280x720, 128x128 window, h=16,
    B refreshed every frame -- every frame's window, lost flag, match count
    and bin set equal to the reference's (track.py:147-205)."""
    f = G.big("cfg3_full")
    vid, _, _ = W.tracking_video()
    assert _digest(vid) == str(f["frames_digest"])
    cx, cy, w, hp = f["win"].tolist()
    rows = gs.track_sequence([gs.Image(v) for v in vid], gs.Window(cx=cx, cy=cy, w=int(w), h_px=int(hp)),
                             gs.ShiftConfig(h=float(f["h"])), [int(f["selected"])], update_bins=True)
    assert [r.window.cx for r in rows] == f["cx"].tolist()
    assert [r.window.cy for r in rows] == f["cy"].tolist()
    assert [r.lost for r in rows] == f["lost"].tolist()
    assert [r.last_match_count for r in rows] == f["matches"].tolist()
    assert [len(r.bins.bins) for r in rows] == f["nbins"].tolist()
    fps = [W.fingerprint(np.array(sorted(r.bins.bins), dtype=np.int64),
                         np.zeros(len(r.bins.bins), dtype=np.int64)) for r in rows]
    assert fps == [int(v) for v in f["bins_fp"]]


@pytest.mark.usefixtures("exact_sums")
@pytest.mark.parametrize("name", ["cfg0"])
def test_big_exact_model_bitwise(name):
    f = G.big(name)
    c = W.CONFIGS[name]
    lab, tr = gs.meanshiftpp(gs.PointSet(W.blobs2d()), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]))
    _check_model(lab, tr, f, c["h"])


@pytest.mark.usefixtures("exact_sums")
@pytest.mark.slow
def test_cfg1_exact_model_bitwise():
    f = G.big("cfg1")
    c = W.CONFIGS["cfg1"]
    lab, tr = gs.segment_pixels(gs.Image(W.cfg1_image()), gs.ShiftConfig(c["h"], c["eta"], c["max_iters"]), "rgb")
    _check_model(lab, tr, f, c["h"])


# ------------------------------------------------- collapsed formulation

@pytest.mark.parametrize("case", ["cloud", "rgb", "rgbxy", "blobs"])
def test_collapsed_mode_bit_identical(case):
    # iterations t >= 1 per run of identical points; the
    # tables / movement are the same exact integers -> identical results
    import torch

    if case == "cloud":
        x, cfg = W.cloud3d(300_000, seed=31).astype(np.float64), gs.ShiftConfig(1.0, 1e-3, 30)
    elif case == "rgb":
        x = gs.image_to_features(gs.Image(W.voronoi_image(400, 300, 20, seed=4)), "rgb").data
        cfg = gs.ShiftConfig(8.0, 1e-3, 100)
    elif case == "rgbxy":
        x = gs.image_to_features(gs.Image(W.voronoi_image(400, 300, 20, seed=5)), "rgbxy", 0.25).data
        cfg = gs.ShiftConfig(10.0, 1e-3, 100)
    else:
        x, cfg = W.blobs2d(100_000, seed=2), gs.ShiftConfig(0.5, 1e-4, 300)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    a, ka, ia, ma, ca = gs.meanshiftpp_device(xd, cfg)
    a = a.cpu().numpy()
    moda = gs.modeseek.last_modes(ka, x.shape[1])
    b, kb, ib, mb, cb = gs.meanshiftpp_device(xd, cfg, collapsed=True)
    b = b.cpu().numpy()
    modb = gs.modeseek.last_modes(kb, x.shape[1])
    assert (ka, ia, ca) == (kb, ib, cb)
    assert np.array_equal(a, b)
    assert np.array_equal(moda, modb)
    np.testing.assert_array_equal(ma, mb)


def test_points_api_float32_equals_pointset_upcast():
    x32 = W.cloud3d(200_000, seed=51)
    cfg = gs.ShiftConfig(1.0, 1e-3, 20)
    a, ta = gs.meanshiftpp_points(x32, cfg)
    b, tb = gs.meanshiftpp(gs.PointSet(x32), cfg)      # PointSet upcasts on the host
    assert np.array_equal(a.labels, b.labels) and np.array_equal(a.modes, b.modes)
    np.testing.assert_array_equal(ta.total_movement_per_iter, tb.total_movement_per_iter)
    bad = x32[:10].copy()
    bad[3, 1] = np.nan
    with pytest.raises(ValueError):
        gs.meanshiftpp_points(bad, cfg)


# ------------------------------------------- streams, in-place accounting

def test_user_stream_and_inplace_accounting():
    # the engine on a caller's (non-default) stream, with the table chain on
    # its side stream, gives the identical result; the in-place shift stores
    # at most the full rewrite, and less once points settle
    import ctypes as C

    import torch

    from paper_2104_00303_b200 import _lib

    x = W.cloud3d(150_000, seed=61).astype(np.float64)
    cfg = gs.ShiftConfig(1.0, 1e-3, 25)
    ref, rtr = gs.meanshiftpp(gs.PointSet(x), cfg)
    xd = torch.from_numpy(x).cuda()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        lab, k, it, mv, conv = gs.meanshiftpp_device(xd, cfg, stream=st.cuda_stream)
    st.synchronize()
    assert np.array_equal(lab.cpu().numpy(), ref.labels) and k == ref.k and it == rtr.iterations
    np.testing.assert_array_equal(mv, rtr.total_movement_per_iter)
    wb = np.zeros(it, dtype=np.uint64)
    _lib.check(_lib.load().gs_fetch_shift_bytes(_lib.context(0), _lib.ptr(wb), C.c_int32(it)))
    full = 8 * 3 * len(x)
    # iteration 0 moves nearly every point (isolated background points are
    # already at their target); no launch stores more than the full rewrite
    assert wb[0] >= full // 2 and np.all(wb <= full + 64)
    assert wb[-1] < wb[0]          # settled points are not rewritten


@pytest.mark.usefixtures("exact_sums")
def test_points_api_sorted_float64_rows():
    # the sort reads fp64 host-layout rows directly (SrcAoS<double>)
    x = W.cloud3d(120_000, seed=62).astype(np.float64)
    cfg = gs.ShiftConfig(1.0, 1e-3, 15)
    a, ta = gs.meanshiftpp_points(x, cfg)
    b = X.meanshiftpp(x, 1.0, 1e-3, 15)
    assert np.array_equal(a.labels, b["labels"]) and np.array_equal(a.modes, b["modes"])
    np.testing.assert_array_equal(ta.total_movement_per_iter, b["movement"])


@pytest.mark.slow
def test_pinned_host_label_delivery_equals_device_labels():
    """A pinned caller buffer of a large run (>= 2^24 points) gets the first
    part of the labels by DMA from the device while host threads expand the
    rest (deliver_labels): identical to the device-written labels, also at an
    offset into the pinned allocation."""
    import torch

    n = (1 << 24) + 12_345
    x = W.cloud3d(n, seed=72)
    cfg = gs.ShiftConfig(1.0, 1e-3, 6)
    dev, k, it, mv, conv = gs.meanshiftpp_device(torch.from_numpy(x).cuda(), cfg)
    dev = dev.cpu().numpy()
    pinned = torch.full((n + 5,), -7, dtype=torch.int64).pin_memory()
    out = pinned.numpy()[5:]
    lab, tr = gs.meanshiftpp_points(x, cfg, labels_out=out)
    assert np.array_equal(out, dev) and lab.k == k and tr.iterations == it
    assert np.all(pinned.numpy()[:5] == -7)
    pageable = np.empty(n, dtype=np.int64)
    gs.meanshiftpp_points(x, cfg, labels_out=pageable)
    assert np.array_equal(pageable, dev)


@pytest.mark.parametrize("iters", [2, 40])
def test_host_label_delivery_equals_device_labels(iters):
    # host entry points on the sorted dense path copy cell0 during the loop
    # and expand per-cell labels on the host threads (gs_engine.cu
    # deliver_labels): identical to the device-written labels, also into an
    # unaligned caller buffer and for runs too short to reach the run-ahead
    # chunks (the copy is then issued after the loop)
    import torch

    x = W.cloud3d(2_500_001, seed=71)
    cfg = gs.ShiftConfig(1.0, 1e-3, iters)
    dev, k, it, mv, conv = gs.meanshiftpp_device(torch.from_numpy(x).cuda(), cfg)
    dev = dev.cpu().numpy()
    a, ta = gs.meanshiftpp_points(x, cfg)
    assert np.array_equal(a.labels, dev) and a.k == k and ta.iterations == it
    big = np.full(len(x) + 3, -7, dtype=np.int64)
    out = big[3:]                       # 24-byte offset: not 64-byte aligned
    b, _ = gs.meanshiftpp_points(x, cfg, labels_out=out)
    assert np.array_equal(out, dev) and np.all(big[:3] == -7)
    import ctypes as C

    from paper_2104_00303_b200 import _lib

    hb, db = C.c_int64(0), C.c_int64(0)
    _lib.check(_lib.load().gs_fetch_transfer_bytes(_lib.context(), _lib.ref(hb), _lib.ref(db)))
    assert hb.value == x.nbytes
    assert 4 * len(x) < db.value < 8 * len(x)     # cell index + per-cell labels + modes
    c, _ = gs.meanshiftpp(gs.PointSet(x), cfg)
    assert np.array_equal(c.labels, dev)
