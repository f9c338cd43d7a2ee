#!/usr/bin/env python
"""MeanShift++ grid shift on B200 -- benchmark (driver contract).

One *step* = one full engine run (modeseek.py:125-146) over one batch of
synthetic input: every grid-shift iteration to convergence / max_iter plus
the device-side label extraction.  Metric: point-updates/s = points x
iterations / seconds (BASELINE.json).  Workload: cfg4 (100M 3-D points,
fp32 input upcast to fp64 iterates, h=1, tol=1e-3, max_iter=50), the largest
configuration and the one the HBM-roofline and scaling targets are judged on.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun, one rank per GPU): the 100M points are sharded by rows and
the per-iteration cell tables are merged with an NCCL all-reduce (strong
scaling, paper_2104_00303_b200/sharded.py).
`--impl reference` times the reference algorithm's CPU restatement
(oracle/, pinned to the reference's outputs) on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2104_00303_b200 import workloads as W  # noqa: E402

METRIC = "point-updates/sec (points x iterations / s)"
UNIT = "point-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=100_000_000, help="points (cfg4 default 1e8)")
    ap.add_argument("--workload", choices=["cfg4", "cfg2"], default="cfg4",
                    help="cfg4 (default, the headline): the 100M-point cloud; cfg2: one 4K RGBxy image per GPU "
                         "(weak scaling, no data-path collective)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-kernels", action="store_true", default=True)
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the row-sharded (NCCL) engine even at one rank (tests the N>1 path)")
    return ap.parse_args()


def cfg4():
    c = W.CONFIGS["cfg4"]
    return c["h"], c["eta"], c["max_iters"]


def workload_config(n, n_gpus):
    h, eta, mi = cfg4()
    return {"workload": f"cfg4: 3-D cloud, n={n:,} fp32 points (fp64 iterates), 50 rotated "
                        f"anisotropic Gaussians + 10% uniform, h={h}, tol={eta}, max_iter={mi}",
            "n": n, "d": 3, "h": h, "tol": eta, "max_iter": mi,
            "sharding": "rows, per-iteration cell-table all-reduce" if n_gpus > 1 else "single GPU",
            "l2": "inputs (1.2 GB fp32 + 2x2.4 GB fp64 iterates) exceed the 126 MB L2"}


# ------------------------------------------------------------- clocks

class Clocks:
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            time.sleep(0.5)           # let the sampler come up before the timed region
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append((time.time(), parts))

    def window(self, t0, t1):
        self.t0, self.t1 = t0, t1

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", 1e30)
        inside = [p for t, p in self.samples if t0 <= t <= t1]
        samples = inside or [p for _, p in self.samples]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.samples = samples
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "in_timed_region": bool(inside)}


# --------------------------------------------------------- CPU baseline

def cpu_sample(n_total, budget_s, x_host=None):
    """Bounded sample of the same workload for the CPU restatement: the first
    1,000,000 rows of the cfg4 input (rows are shuffled, so this is a uniform
    random subsample) when the full input is at hand, else the cfg4 generator
    at n=1,000,000; iteration cap sized to the time budget (~0.45 s/iter)."""
    n = min(1_000_000, n_total)
    iters = int(max(1, min(50, budget_s / 0.45)))
    if x_host is not None:
        return x_host[:n].astype(np.float64), iters, f"cfg4 input rows [0, {n:,})"
    return W.cloud3d(n, seed=4).astype(np.float64), iters, f"cfg4 generator at n={n:,} (seed 4)"


def run_oracle(x, iters):
    from oracle import gridshift_oracle as O

    h, eta, _ = cfg4()
    t0 = time.perf_counter()
    r = O.meanshiftpp(x, h, eta, iters)
    dt = time.perf_counter() - t0
    return x.shape[0] * r["iterations"], dt, r["iterations"]


def host_cpu():
    """Host CPU model and logical core count."""
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count()}


def reference_engine():
    """The unmodified reference engine from the reference install
    (baseline/_ref, scripts/install_reference.sh), else None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "gridshift" / "modeseek.py").exists():
        return None
    sys.path.insert(0, str(ref))
    try:
        import gridshift.modeseek as rms
        from gridshift.grid import PointSet as RPointSet
    except Exception:   # noqa: BLE001 -- a broken install falls back to the port
        return None
    if getattr(rms.ENGINES["meanshiftpp"], "__gridshift_b200__", False):
        return None     # patched by install(): not the reference's code path
    return rms, RPointSet


def run_reference_engine(x, iters, eng):
    """ENGINES["meanshiftpp"](PointSet, ShiftConfig) of the reference itself
    (modeseek.py:125,288), timed around the engine call only (its bench.py:44-51)."""
    rms, RPointSet = eng
    h, eta, _ = cfg4()
    pts = RPointSet(x)
    t0 = time.perf_counter()
    _, tr = rms.ENGINES["meanshiftpp"](pts, rms.ShiftConfig(h=h, eta=eta, max_iters=iters))
    dt = time.perf_counter() - t0
    return x.shape[0] * tr.iterations, dt, tr.iterations


def reference_arm(a):
    """The reference's own CPU implementation on this host (rank 0 only):
    the unmodified gridshift engine from baseline/_ref when installed
    ("kind": "reference"), else its pinned numpy restatement ("port").
    Each step is one engine call on a bounded sample of the cfg4 workload
    (first 1M rows of the real input, iteration-capped), stated in
    `reference_sample`; the metric is a rate, so the sample is comparable."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget = max(5.0, 150.0 / max(1, a.steps + a.warmup))
    x_full = W.cloud3d(a.n)
    x, iters, what = cpu_sample(a.n, budget, x_full)
    del x_full
    eng = reference_engine()
    run = (lambda: run_reference_engine(x, iters, eng)) if eng else (lambda: run_oracle(x, iters))
    for _ in range(a.warmup):
        run()
    ups, secs, it = 0, 0.0, 0
    for _ in range(a.steps):
        u, dt, it = run()
        ups += u
        secs += dt
    v = ups / secs
    kind = "reference" if eng else "port"
    impl = ("gridshift.modeseek.ENGINES['meanshiftpp'] from baseline/_ref (unmodified reference)"
            if eng else "oracle/gridshift_oracle.py (numpy restatement, bitwise-pinned to the reference)")
    sample = f"{what} (uniform random subsample), {it} iterations per step (max_iter cap), h=1, tol=1e-3"
    cfg = workload_config(a.n, 1)
    cfg["reference_sample"] = {"rows": int(x.shape[0]), "iterations_per_step": int(it),
                               "of": f"the cfg4 input (n={a.n:,}); value is the sample's point-updates/s"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * secs / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded numpy, paper_2104_00303_b200/workloads.py)",
            "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample,
                             "implementation": impl, "host_cpu": host_cpu(),
                             "note": "the reference path is single-threaded numpy (unique/bincount/"
                                     "searchsorted do not thread): 1 core"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- our arm

def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel):
    """Mean per-launch DRAM bytes of `kernel` over a whole engine run, from the
    committed ncu capture profiles/<kernel>_traffic_r*.csv (all launches of
    one run), else the --set full summary profiles/ncu_full_*.json."""
    import csv as _csv

    for f in sorted((ROOT / "profiles").glob("*_traffic_r*.csv"), reverse=True):
        vals = {}
        for r in _csv.reader(f.read_text().splitlines()):
            if len(r) > 12 and kernel in r[4] and r[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[-2], 1.0)
                vals[r[0]] = vals.get(r[0], 0.0) + float(r[-1].replace(",", "")) * scale
        if vals:
            return sum(vals.values()) / len(vals), f.name
    for f in sorted((ROOT / "profiles").glob("ncu_full_*.json"), reverse=True):
        try:
            d = json.loads(f.read_text())
        except ValueError:
            continue
        k = d.get("kernels", {}).get(kernel)
        if k and k.get("dram_bytes") is not None:
            return float(k["dram_bytes"]), f.name
    return None, None


def our_arm(a):
    import torch
    import torch.distributed as dist

    import paper_2104_00303_b200 as gs
    from paper_2104_00303_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["GRIDSHIFT_DEVICE"] = str(local)
    shard = world > 1 or a.force_sharded
    if shard:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h, eta, mi = cfg4()
    n = a.n
    x_host = W.cloud3d(n)                       # fp32 (n, 3), seeded
    if shard:
        from paper_2104_00303_b200 import sharded

        lo, hi = sharded.shard_bounds(n, world, rank)
        x_dev = torch.from_numpy(x_host[lo:hi]).cuda()
    else:
        lo, hi = 0, n
        x_dev = torch.from_numpy(x_host).cuda()
    cfg = gs.ShiftConfig(h=h, eta=eta, max_iters=mi)
    labels = torch.empty(x_dev.shape[0], dtype=torch.int64, device="cuda")

    last = {}

    def step():
        if shard:
            return sharded.meanshiftpp_sharded(x_dev, cfg, labels, n_total=n)
        _, k, it, mv, conv = gs.meanshiftpp_device(x_dev, cfg, labels)
        last["k"] = k
        return it

    def barrier():
        if shard:
            dist.barrier()

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    _lib.profile(1)
    iters_total = 0
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record()
        for _ in range(a.steps):
            iters_total += step()
        e1.record()
        torch.cuda.synchronize()
        clk.window(w0, time.time())
        barrier()
    ms = e0.elapsed_time(e1)
    if not shard:   # sanity (untimed): labels dense in [0, k)
        u = torch.unique(labels)
        assert int(u[0]) == 0 and int(u[-1]) == last["k"] - 1 and u.numel() == last["k"], "bad labels"
    prof = _lib.profile(2)
    _lib.profile(0)
    # bytes k_shift actually stored per iteration of the last run (in-place
    # iterate, unchanged coordinate pairs are not rewritten)
    import ctypes as _C
    last_iters = iters_total // a.steps
    wb = np.zeros(max(1, last_iters), dtype=np.uint64)
    _lib.check(_lib.load().gs_fetch_shift_bytes(_lib.context(local), _lib.ptr(wb), _C.c_int32(last_iters)))
    stored_per_launch = float(wb[:last_iters].mean()) if last_iters else 0.0
    if shard:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    per_step_iters = iters_total / a.steps
    value = n * iters_total / (ms / 1e3)

    # roofline of the dominant per-point kernel
    n_local = x_dev.shape[0]
    d = 3
    # k_shift reads y and writes y' (16*d B/point); k_hist bins the input
    # once per step (later tables are derived per cell, k_derive)
    # k_shift: reads y (8*d B/point) and stores the coordinate pairs that
    # changed (at most 8*d B/point; counted on device, gs_fetch_shift_bytes)
    bytes_per = {"hist": 8 * d * n_local, "shift": 8 * d * n_local + stored_per_launch}
    work = {"hist": a.steps, "shift": iters_total}
    # per-point kernels only: the table chain (agg, derive) runs on a side
    # stream overlapping the shifts, so its event spans include waiting
    kern = max(("hist", "shift"), key=lambda k: prof[k][0])
    peak, peak_src = measured_peak()
    roof = None
    if kern in bytes_per:
        alg = bytes_per[kern] * work[kern]
        achieved = alg / (prof[kern][0] / 1e3) / 1e9
        traffic, tsrc = ncu_traffic("k_shift_tma" if kern == "shift" else f"k_{kern}")
        roof = {"kernel": "k_shift_tma" if kern == "shift" else f"k_{kern}", "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": bytes_per[kern],
                "bytes_note": ("k_shift: 8*d*n read + the bytes actually stored (in-place iterate; bitwise-"
                               "unchanged coordinate pairs are not rewritten); the full rewrite would be "
                               f"16*d*n = {16 * d * n_local} B") if kern == "shift" else None,
                "avg_launch_ms": prof[kern][0] / work[kern], "traffic_source": tsrc}
        if kern == "shift":
            # the same launch time against SURVEY 8(d)'s full-rewrite bytes
            # (16*d*n per launch); > 1 is possible only because unchanged
            # coordinate pairs are not stored
            roof["frac_s8d"] = 16 * d * n_local / (roof["avg_launch_ms"] / 1e3) / 1e9 / peak
    kernels = {k: {"ms": v[0], "launches": v[1]} for k, v in prof.items() if v[1]}
    for k in ("hist", "shift"):
        if k in kernels and prof[k][0] > 0:
            kernels[k]["achieved_gbs"] = bytes_per[k] * work[k] / (prof[k][0] / 1e3) / 1e9
    launches = int(sum(v[1] for v in prof.values()))
    # the histogram kernel's own roofline (north_star: shift and histogram
    # each against the HBM peak); one launch per step, on the input
    roof_hist = None
    if prof["hist"][1] and prof["hist"][0] > 0:
        ach = bytes_per["hist"] * work["hist"] / (prof["hist"][0] / 1e3) / 1e9
        tr, tsrc = ncu_traffic("k_hist")
        roof_hist = {"kernel": "k_hist", "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": tr, "peak_source": peak_src,
                     "alg_bytes_per_launch": bytes_per["hist"],
                     "bytes_note": "k_hist: reads the sorted fp64 iterate once, 8*d*n B",
                     "avg_launch_ms": prof["hist"][0] / work["hist"], "traffic_source": tsrc}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": max(3, a.warmup), "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded numpy, paper_2104_00303_b200/workloads.py); fp32 input upcast "
                    "on device like PointSet (grid.py:43)",
            "config": workload_config(n, world), "iterations_per_step": per_step_iters,
            "roofline": roof, "roofline_hist": roof_hist, "kernels": kernels,
            "kernels_note": "CUDA-event spans per kind over the timed region; agg/derive run on a "
                            "low-priority side stream concurrently with the shifts (their spans include "
                            "waiting for SM slots); see profiles/launches_r02_summary.json for serialised "
                            "per-kernel device time",
            "gpu_launches": launches, "clocks": clk.summary(),
            "byte_model": {
                "executed": "per run: 1 per-point histogram pass (k_hist, 8*d*n B) on the sorted input; "
                            "per iteration: 1 per-point shift (8*d*n B read + the changed 16-B coordinate "
                            "pairs stored) + the O(cells) table chain (aggregate -> derive: table t+1 is "
                            "derived per cell from table t, so points are not re-binned)",
                "hist_passes_per_run": 1,
                "shift_stored_bytes_per_iter_mean": stored_per_launch,
                "shift_full_rewrite_bytes_per_iter": 16 * d * n_local,
                "s8d_bytes_per_step": per_step_iters * 24 * d * n_local,
                "s8d_step_frac": (per_step_iters * 24 * d * n_local) / (ms / a.steps / 1e3) / 1e9 / peak,
                "note": "SURVEY 8(d) counts 24*d*n B per iteration (re-bin + full rewrite); s8d_step_frac is "
                        "that byte count over the measured step time against the peak, > 1 because the "
                        "engine does less work than 8(d) assumes, with bit-identical results"}}

    if shard:
        line["config"]["parallelism"] = f"rows sharded over {world} GPU(s), NCCL"
    if rank == 0 and not shard:
        line["sum_order"] = ("seqmodel (default): the reference's sequential per-cell sums (np.bincount, "
                             "grid.py:186-187) without the point order -- single-source cells by the closed "
                             "form (bit for bit), mixed cells folded from their sources in proportion per "
                             "binade; cells, counts and labels equal the reference's, modes within 1.5e-11*h "
                             "on this workload (tests/test_gpu_parity.py::test_cfg4_100m_vs_reference)")
        line["refsum"] = refsum_stats(gs, last_iters)
        line["reference_order"] = order_leg(gs, torch, x_dev, cfg, labels, n, a.steps, "reference")
        line["exact_order"] = order_leg(gs, torch, x_dev, cfg, labels, n, a.steps, "exact")
        line["collapsed"] = collapsed_leg(gs, torch, x_dev, cfg, labels, n, a.steps)
    if not a.no_e2e:
        if shard:
            e = e2e_sharded(sharded, dist, torch, x_host[lo:hi], cfg, n, min(a.steps, 3))
            if rank == 0:
                line["e2e"] = e
        elif rank == 0:
            line["e2e"] = e2e(x_host, cfg, n, min(a.steps, 3))
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        x, iters, what = cpu_sample(n, 12.0, x_host)
        eng = reference_engine()
        ups, secs, it = run_reference_engine(x, iters, eng) if eng else run_oracle(x, iters)
        line["cpu_baseline"] = {"value": ups / secs, "unit": UNIT, "cores": 1,
                                "kind": "reference" if eng else "port",
                                "sample": f"{what} (uniform random subsample), {it} iterations, " +
                                          ("the unmodified reference engine (baseline/_ref)" if eng else
                                           "oracle/gridshift_oracle.py (numpy, single-threaded)"),
                                "host_cpu": host_cpu()}
    if shard:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def cfg2_arm(a):
    """cfg2 (BASELINE configs[2]): a batch of 3840x2160 RGB+xy images, one per
    GPU (rank r segments image r; no collective on the data path,
    cli.py:206-216).  `value`: features resident in HBM, the engine run only;
    `e2e`: segment_image with uint8 host pixels (fused features, labels and
    mean colours back on the host)."""
    import torch
    import torch.distributed as dist

    import paper_2104_00303_b200 as gs
    from paper_2104_00303_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["GRIDSHIFT_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = W.CONFIGS["cfg2"]
    cfg = gs.ShiftConfig(c["h"], c["eta"], c["max_iters"])
    img = gs.Image(W.cfg2_image(rank % 8))
    x = gs.image_to_features(img, "rgbxy", 0.25).data
    n, d = x.shape
    x_dev = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    labels = torch.empty(n, dtype=torch.int64, device="cuda")

    def step():
        return gs.meanshiftpp_device(x_dev, cfg, labels)[2]

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    _lib.profile(1)
    iters_total = 0
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record()
        for _ in range(a.steps):
            iters_total += step()
        e1.record()
        torch.cuda.synchronize()
        clk.window(w0, time.time())
        barrier()
    ms = e0.elapsed_time(e1)
    prof = _lib.profile(2)
    _lib.profile(0)
    # end to end: uint8 pixels from pinned host memory, labels + mean colours back
    pix = torch.empty(img.pixels.shape, dtype=torch.uint8, pin_memory=True).numpy()
    pix[:] = img.pixels
    himg = gs.Image(pix)
    gs.segment_image(himg, cfg, "rgbxy", scale=0.25)
    esteps = min(a.steps, 5)
    barrier()
    t0 = time.perf_counter()
    eit = 0
    for _ in range(esteps):
        seg, tr = gs.segment_image(himg, cfg, "rgbxy", scale=0.25)
        eit += tr.iterations
    esecs = time.perf_counter() - t0
    import ctypes as C

    hb, db = C.c_int64(0), C.c_int64(0)
    _lib.check(_lib.load().gs_fetch_transfer_bytes(_lib.context(local), _lib.ref(hb), _lib.ref(db)))
    tot_iters, e_ups = iters_total, n * eit
    if world > 1:
        t = torch.tensor([ms, esecs], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, esecs = float(t[0]), float(t[1])
        u = torch.tensor([iters_total, n * eit], dtype=torch.float64, device="cuda")
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        tot_iters, e_ups = float(u[0]), float(u[1])
    peak, peak_src = measured_peak()
    kernels = {k: {"ms": v[0], "launches": v[1]} for k, v in prof.items() if v[1]}
    roofs = {}
    # live launches: one histogram per run; one shift per iteration (the loop
    # enqueues chunks ahead, launches past the stop flag exit at once)
    live = {"hist": a.steps, "shift": iters_total}
    for kind, per_launch in (("hist", 8 * d * n), ("shift", 16 * d * n)):
        if prof[kind][1] and prof[kind][0] > 0:
            ach = per_launch * live[kind] / (prof[kind][0] / 1e3) / 1e9
            roofs[kind] = {"kernel": "k_hist" if kind == "hist" else "k_shift", "bound": "hbm", "achieved": ach,
                           "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None,
                           "peak_source": peak_src, "alg_bytes_per_launch": per_launch,
                           "avg_launch_ms": prof[kind][0] / live[kind],
                           "bytes_note": ("8*d*n B read per launch" if kind == "hist" else
                                          "16*d*n B per launch (read y, write y'; SURVEY 8d)")}
    line = {"metric": METRIC, "value": n * tot_iters / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": max(3, a.warmup), "ms_per_step": ms / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Voronoi image, paper_2104_00303_b200/workloads.py)",
            "config": {"workload": f"cfg2: one 3840x2160 RGB+xy image per GPU (n={n:,} fp64 points, d=5, "
                                   f"h={c['h']}, tol={c['eta']}, max_iter={c['max_iters']}, scale=0.25), "
                                   "sparse 5-D lattice (hash tables)",
                       "n_per_gpu": n, "d": d, "h": c["h"], "tol": c["eta"], "max_iter": c["max_iters"],
                       "sharding": "one image per rank, no data-path collective",
                       "l2": "the iterate (2 x 332 MB fp64) exceeds the 126 MB L2"},
            "iterations_per_step": iters_total / a.steps, "roofline": roofs.get("shift"),
            "roofline_hist": roofs.get("hist"), "kernels": kernels,
            "gpu_launches": int(sum(v[1] for v in prof.values())), "clocks": clk.summary(),
            "e2e": {"value": e_ups / esecs, "unit": UNIT, "h2d_bytes_per_step": int(hb.value),
                    "d2h_bytes_per_step": int(db.value), "steps": esteps,
                    "api": "paper_2104_00303_b200.segment_image(Image uint8 (2160, 3840, 3), ShiftConfig, "
                           "'rgbxy', scale=0.25) -> gs_segment_image (C ABI)"}}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def refsum_stats(gs, iters):
    """Per-table counters of the reference-order sums in the last timed run."""
    st = gs.modeseek.last_refsum_stats(iters)
    return {"mixed_cells_per_table": [int(v) for v in st[:, 0]],
            "points_through_global_sort_per_table": [int(v) for v in st[:, 2]],
            "longest_mixed_cell_per_table": [int(v) for v in st[:, 3]],
            "note": "per table: cells that received several source cells (folded by the sequential model in "
                    "the default order; in point-index order under GS_SUMS_REFERENCE, where the second "
                    "list counts the points that go through the global radix sort); single-source cells "
                    "use the closed form per binade"}


ORDER_NOTES = {
    "reference": "GS_SUMS_REFERENCE: every mixed cell summed in point-index order (index-ordered point lists, "
                 "radix sort for long cells); every iterate equals the reference's bit for bit",
    "exact": "GS_SUMS_EXACT: exact fixed-point sums rounded once (order-independent; the row-sharded multi-GPU "
             "path computes these); modes 1.1e-8*h from the reference's on this workload, over the 1e-9*h bar, "
             "so not the headline",
}


def order_leg(gs, torch, x_dev, cfg, labels, n, steps, order):
    """Same workload under another sum order."""
    with gs.sum_order(order):
        gs.meanshiftpp_device(x_dev, cfg, labels)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        it = 0
        e0.record()
        for _ in range(steps):
            it += gs.meanshiftpp_device(x_dev, cfg, labels)[2]
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"value": n * it / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "note": ORDER_NOTES[order]}


def collapsed_leg(gs, torch, x_dev, cfg, labels, n, steps):
    """Same workload, iterations t >= 1 in the collapsed-group formulation
    (SURVEY 8f rank 1): bit-identical results, but iterations move one
    position per run of identical points instead of every point -- reported
    beside, never as, the per-point metric."""
    gs.meanshiftpp_device(x_dev, cfg, labels, collapsed=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    it = 0
    e0.record()
    for _ in range(steps):
        it += gs.meanshiftpp_device(x_dev, cfg, labels, collapsed=True)[2]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"value": n * it / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps,
            "note": "collapsed-group formulation (SURVEY.md 8f rank 1): after iteration 0 each run of "
                    "identical points moves as one; results bit-identical to the per-point engine "
                    "(tests/test_gpu_parity.py::test_collapsed_mode_bit_identical); not a per-point "
                    "workload, so not the headline"}


def e2e_sharded(sharded, dist, torch, x_shard, cfg, n, steps):
    """N-GPU end to end through the sharded public entry: every step copies
    this rank's rows (fp64, pinned host) to its GPU, runs the sharded engine
    and copies its labels back; time = max over ranks."""
    pts = torch.empty((x_shard.shape[0], 3), dtype=torch.float64, pin_memory=True)
    pts.numpy()[:] = x_shard
    lab_host = torch.empty(x_shard.shape[0], dtype=torch.int64, pin_memory=True)
    x_dev = torch.empty_like(pts, device="cuda")
    labels = torch.empty(x_shard.shape[0], dtype=torch.int64, device="cuda")

    def one():
        x_dev.copy_(pts, non_blocking=True)
        it = sharded.meanshiftpp_sharded(x_dev, cfg, labels, n_total=n)
        lab_host.copy_(labels, non_blocking=True)
        torch.cuda.synchronize()
        return it

    one()
    dist.barrier()
    t0 = time.perf_counter()
    it = sum(one() for _ in range(steps))
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    secs = float(dt.item())
    return {"value": n * it / secs, "unit": UNIT, "h2d_bytes_per_step": int(pts.numel() * 8),
            "d2h_bytes_per_step": int(lab_host.numel() * 8), "steps": steps,
            "api": "paper_2104_00303_b200.sharded.meanshiftpp_sharded (per-rank H2D/D2H, max over ranks)"}


def e2e(x_host, cfg, n, steps):
    """Public host API with the input in pinned host memory: every step copies
    the points host->device and the labels (+ modes) device->host inside the
    timed region.  cfg4's points are float32 (BASELINE config), so they cross
    PCIe as float32 through meanshiftpp_points and are upcast on device,
    bit-identical to PointSet's host upcast (grid.py:43)."""
    import torch

    import paper_2104_00303_b200 as gs

    pts = torch.empty((n, 3), dtype=torch.float32, pin_memory=True).numpy()
    pts[:] = x_host
    lab_out = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
    gs.meanshiftpp_points(pts, cfg, labels_out=lab_out)     # warm
    ups = 0
    k = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        lab, tr = gs.meanshiftpp_points(pts, cfg, labels_out=lab_out)
        ups += n * tr.iterations
        k = lab.k
    dt = time.perf_counter() - t0
    # bytes the last call moved, as the library counted them: the fp32 rows
    # up; down the per-point initial-cell index (copied while the loop runs)
    # + per-cell labels, expanded into lab_out by host threads (sorted dense
    # path), or the int64 labels otherwise; + the modes
    import ctypes as C

    from paper_2104_00303_b200 import _lib

    hb, db = C.c_int64(0), C.c_int64(0)
    _lib.check(_lib.load().gs_fetch_transfer_bytes(_lib.context(), _lib.ref(hb), _lib.ref(db)))
    assert hb.value == pts.nbytes, (hb.value, pts.nbytes)
    return {"value": ups / dt, "unit": UNIT, "h2d_bytes_per_step": int(hb.value),
            "d2h_bytes_per_step": int(db.value), "steps": steps,
            "labels": "int64 into the caller's pinned buffer; the sorted dense path sends 4 B/point of "
                      "initial-cell index during the loop + 4 B/cell of labels; host threads expand 60% of the "
                      "labels from them while the device writes the other 40% into the pinned buffer by DMA",
            "api": "paper_2104_00303_b200.meanshiftpp_points(float32 (n,3), ShiftConfig) -> "
                   "gs_meanshiftpp_host (C ABI)"}


def main():
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
    elif a.workload == "cfg2":
        cfg2_arm(a)
    else:
        our_arm(a)


if __name__ == "__main__":
    main()
