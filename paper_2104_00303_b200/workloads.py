"""Seeded synthetic inputs for the five BASELINE.json configurations.

BASELINE.json names no public dataset, so every input is generated here
with numpy's `default_rng` (identical bits on every host running the same
numpy).  None of these generators exist in the reference; cfg0 follows the
shape of `gridshift.data.generate_mixture` (data.py:58-66).

    cfg0  2-D Gaussian blobs            n=100,000      h=0.5  tol=1e-4 max=300
    cfg1  RGB Voronoi 1920x1080 (64)    n=2,073,600    h=8    tol=1e-3 max=100
    cfg2  RGBxy Voronoi 3840x2160 (256) n=8,294,400/img h=10  tol=1e-3 max=100 (assumed)
    cfg3  tracking video 300x1280x720   window 128x128 h=16 (colour)
    cfg4  3-D cloud                      n=100,000,000  h=1    tol=1e-3 max=50
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    "cfg0": dict(h=0.5, eta=1e-4, max_iters=300),
    "cfg1": dict(h=8.0, eta=1e-3, max_iters=100),
    "cfg2": dict(h=10.0, eta=1e-3, max_iters=100),
    "cfg3": dict(h=16.0),
    "cfg4": dict(h=1.0, eta=1e-3, max_iters=50),
}


def blobs2d(n: int = 100_000, seed: int = 0) -> np.ndarray:
    """cfg0: 5 isotropic Gaussians (sigma 0.4), centres ~U[0,10]^2, equal weights."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 10.0, size=(5, 2))
    comp = rng.choice(5, size=n)
    return centres[comp] + rng.normal(0.0, 0.4, size=(n, 2))


def voronoi_image(width: int, height: int, sites: int, seed: int,
                  noise: float = 8.0) -> np.ndarray:
    """cfg1/cfg2: Voronoi partition of seeded sites, uniform colour per region,
    i.i.d. N(0, noise^2) per channel, rounded half-up and clipped to uint8."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = np.column_stack([rng.uniform(0, width, sites), rng.uniform(0, height, sites)])
    colours = rng.uniform(0.0, 255.0, size=(sites, 3))
    tree = cKDTree(pts)
    out = np.empty((height, width, 3), dtype=np.uint8)
    xs = np.arange(width, dtype=np.float64) + 0.5
    band = max(1, (1 << 22) // width)
    for y0 in range(0, height, band):
        y1 = min(height, y0 + band)
        gy, gx = np.meshgrid(np.arange(y0, y1, dtype=np.float64) + 0.5, xs, indexing="ij")
        _, owner = tree.query(np.column_stack([gx.ravel(), gy.ravel()]))
        base = colours[owner] + rng.normal(0.0, noise, size=(owner.size, 3))
        out[y0:y1] = np.clip(np.floor(base + 0.5), 0, 255).astype(np.uint8).reshape(y1 - y0, width, 3)
    return out


def cfg1_image(seed: int = 1) -> np.ndarray:
    return voronoi_image(1920, 1080, 64, seed)


def cfg2_image(index: int = 0) -> np.ndarray:
    return voronoi_image(3840, 2160, 256, 100 + index)


def cloud3d(n: int = 100_000_000, seed: int = 4, k: int = 50,
            dtype=np.float32) -> np.ndarray:
    """cfg4: 90% from k anisotropic rotated Gaussians (axis sigma ~U[0.1,1],
    centres ~U[0,100]^3), 10% uniform background in [0,100]^3; the rows are
    shuffled with a seeded permutation so contiguous shards are balanced."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 100.0, size=(k, 3))
    sig = rng.uniform(0.1, 1.0, size=(k, 3))
    rot = np.stack([np.linalg.qr(rng.normal(size=(3, 3)))[0] for _ in range(k)])
    n_fg = (n * 9) // 10
    out = np.empty((n, 3), dtype=dtype)
    step = 1 << 23
    for a in range(0, n_fg, step):
        b = min(n_fg, a + step)
        comp = rng.integers(0, k, size=b - a)
        z = rng.normal(size=(b - a, 3)) * sig[comp]
        out[a:b] = centres[comp] + np.einsum("nij,nj->ni", rot[comp], z)
    out[n_fg:] = rng.uniform(0.0, 100.0, size=(n - n_fg, 3))
    perm = rng.permutation(n)
    return out[perm]


# ------------------------------------------------------------ cfg3 video

def _value_noise(rng, width, height, cell=40, octaves=3):
    """Smooth Perlin-style texture: bilinearly upsampled random lattices summed
    over octaves, mapped into [40, 200]."""
    acc = np.zeros((height, width))
    amp, total = 1.0, 0.0
    for o in range(octaves):
        c = max(2, cell >> o)
        gh, gw = height // c + 2, width // c + 2
        lat = rng.uniform(0.0, 1.0, size=(gh, gw))
        yy = np.arange(height) / c
        xx = np.arange(width) / c
        y0 = yy.astype(int)
        x0 = xx.astype(int)
        fy = (yy - y0)[:, None]
        fx = (xx - x0)[None, :]
        fy = fy * fy * (3 - 2 * fy)
        fx = fx * fx * (3 - 2 * fx)
        a = lat[y0][:, x0]
        b = lat[y0][:, x0 + 1]
        c_ = lat[y0 + 1][:, x0]
        d = lat[y0 + 1][:, x0 + 1]
        acc += amp * ((a * (1 - fx) + b * fx) * (1 - fy) + (c_ * (1 - fx) + d * fx) * fy)
        total += amp
        amp *= 0.5
    return 40.0 + 160.0 * acc / total


def tracking_video(n_frames: int = 300, width: int = 1280, height: int = 720,
                   seed: int = 3, axes=(60, 40)):
    """cfg3: an ellipse (semi-axes 60x40 px) with per-pixel colour ~N(mu, 6^2)
    following a seeded smooth path over a value-noise background, with a
    global brightness drift x(1 + 0.002 t).  Returns (frames uint8
    (T,H,W,3), centres (T,2) float64, object colour mu)."""
    rng = np.random.default_rng(seed)
    bg = np.stack([_value_noise(rng, width, height) for _ in range(3)], axis=-1)
    # object colour well away from the background palette [40, 200]
    mu = np.array([235.0, 20.0, 225.0])
    ax, ay = axes
    # smooth path: sum of low-frequency sinusoids, kept inside the frame
    t = np.arange(n_frames, dtype=np.float64)
    ph = rng.uniform(0, 2 * np.pi, size=4)
    cx = width / 2 + (width / 2 - ax - 80) * (0.7 * np.sin(2 * np.pi * t / 400 + ph[0])
                                              + 0.3 * np.sin(2 * np.pi * t / 170 + ph[1]))
    cy = height / 2 + (height / 2 - ay - 80) * (0.7 * np.sin(2 * np.pi * t / 330 + ph[2])
                                                + 0.3 * np.sin(2 * np.pi * t / 140 + ph[3]))
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float64)
    frames = np.empty((n_frames, height, width, 3), dtype=np.uint8)
    for i in range(n_frames):
        f = bg.copy()
        inside = ((xx - cx[i]) / ax) ** 2 + ((yy - cy[i]) / ay) ** 2 <= 1.0
        m = int(inside.sum())
        f[inside] = mu + rng.normal(0.0, 6.0, size=(m, 3))
        f *= 1.0 + 0.002 * i
        frames[i] = np.clip(np.floor(f + 0.5), 0, 255).astype(np.uint8)
    return frames, np.column_stack([cx, cy]), mu


def fingerprint(cells: np.ndarray, counts: np.ndarray) -> int:
    """Order-independent 64-bit fingerprint of a cell table {(cell, count)}.

    sum over cells of splitmix64-chained hashes, mod 2^64.  The CUDA engine
    computes the same value on device for every iteration's table, so one
    integer pins the whole (cells, counts) pair bit for bit.
    """
    cells = np.asarray(cells, dtype=np.int64)
    counts = np.asarray(counts, dtype=np.int64)
    k, d = cells.shape
    with np.errstate(over="ignore"):
        x = np.full(k, (0x9E3779B97F4A7C15 * (d + 1)) & 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
        for j in range(d):
            x = _mix64(x ^ cells[:, j].view(np.uint64))
        x = _mix64(x ^ counts.view(np.uint64))
        return int(x.sum(dtype=np.uint64))


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))
