"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference's phantoms (geometry.py:142-247) do not cover BASELINE's
scenes, so these generators are builder-defined.  Every draw
comes from ``numpy.random.default_rng(seed)`` in a fixed order and every
float input is quantised to float32, so the CPU oracle and the GPU consume
bit-identical values.  Choices BASELINE leaves open are fixed here and in
DESIGN.md:

* config 1: a0 ~ lognormal with ARITHMETIC mean 0.2 mm, sigma_log 0.3,
  clipped to [0.1, 0.4] mm; target = forward(mu + N(0, 0.05 mm)).
* tubes / trees: random-walk polylines (0.5 mm steps, reflected into the
  cube); ball centres uniform along the centreline plus a uniform-disc offset
  inside the tube; a0 = 0.5 * tube radius * U(0.8, 1.2).
* hemispheres: ``fibonacci_sphere(2M, r)[:M]`` (the reference lattice,
  geometry.py:22-37, whose z decreases with index); radius 40 mm (configs 2,
  5) or 60 mm (configs 3, 4).
* motion: radial pulsation s_k = 1 + 0.08 sin(2 pi k / 8) about each ball's
  centreline point (offset and a0 scale with s_k) plus a sinusoidal drift
  d_k = 0.5 mm * (sin(2 pi k / 8), 0.5 sin(4 pi k / 8), 0).
* model: poly+Fourier basis (N = 8), multiplicative coordinates, baseline =
  frame-0 ground truth, omega ~ U(-0.01, 0.01).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import (DynamicCloud, ReconConfig, SensorArray,
                   default_basis_grid, frame_times)

GOLDEN_RATIO = (1.0 + np.sqrt(5.0)) / 2.0


def q32(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def fibonacci_sphere(m: int, radius: float) -> np.ndarray:
    """Golden-angle lattice (same closed form as geometry.py:22-37)."""
    i = np.arange(m, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / m
    phi = 2.0 * np.pi * i * (1.0 - 1.0 / GOLDEN_RATIO)
    s = np.sqrt(1.0 - z * z)
    return radius * np.column_stack([s * np.cos(phi), s * np.sin(phi), z])


def hemisphere(m: int, radius: float) -> np.ndarray:
    return fibonacci_sphere(2 * m, radius)[:m]


def planar_grid(n: int, pitch: float) -> np.ndarray:
    ix, iy = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    c = (n - 1) / 2.0
    return np.column_stack([(ix.ravel() - c) * pitch, (iy.ravel() - c) * pitch,
                            np.zeros(n * n)])


def _random_walk(rng, start, direction, length, half, step=0.5, turn=0.25):
    n = max(2, int(round(length / step)) + 1)
    pts = np.empty((n, 3))
    pts[0] = start
    d = direction / np.linalg.norm(direction)
    for k in range(1, n):
        d = d + turn * rng.normal(size=3)
        d /= np.linalg.norm(d)
        p = pts[k - 1] + step * d
        for ax in range(3):                       # reflect into the cube
            if abs(p[ax]) > half:
                p[ax] = np.sign(p[ax]) * (2 * half - abs(p[ax]))
                d[ax] = -d[ax]
        pts[k] = p
    return pts


def _balls_on_polylines(rng, lines, radii, counts, a0_scale=0.5):
    """Centres along each polyline + uniform-disc offsets inside the tube."""
    mus, a0s, axes = [], [], []
    for pts, r, n in zip(lines, radii, counts):
        seg = np.diff(pts, axis=0)
        seglen = np.linalg.norm(seg, axis=1)
        cum = np.concatenate([[0.0], np.cumsum(seglen)])
        s = rng.uniform(0.0, cum[-1], n)
        k = np.clip(np.searchsorted(cum, s, side="right") - 1, 0,
                    len(seg) - 1)
        frac = (s - cum[k]) / np.maximum(seglen[k], 1e-12)
        axis_pt = pts[k] + frac[:, None] * seg[k]
        tdir = seg[k] / np.maximum(seglen[k], 1e-12)[:, None]
        # orthonormal frame around the tangent
        ref = np.where(np.abs(tdir[:, :1]) < 0.9, np.array([[1.0, 0, 0]]),
                       np.array([[0, 1.0, 0]]))
        u = np.cross(tdir, ref)
        u /= np.linalg.norm(u, axis=1)[:, None]
        w = np.cross(tdir, u)
        rad = r * np.sqrt(rng.uniform(0, 1, n))
        ang = rng.uniform(0, 2 * np.pi, n)
        off = rad[:, None] * (np.cos(ang)[:, None] * u + np.sin(ang)[:, None] * w)
        mus.append(axis_pt + off)
        axes.append(axis_pt)
        a0s.append(a0_scale * r * rng.uniform(0.8, 1.2, n))
    return np.concatenate(mus), np.concatenate(a0s), np.concatenate(axes)


def tubes(rng, n_balls, n_tubes, length, r_lo, r_hi, half):
    lines, radii = [], []
    for _ in range(n_tubes):
        start = rng.uniform(-0.6 * half, 0.6 * half, 3)
        lines.append(_random_walk(rng, start, rng.normal(size=3), length,
                                  half))
        radii.append(rng.uniform(r_lo, r_hi))
    counts = np.full(n_tubes, n_balls // n_tubes)
    counts[: n_balls - counts.sum()] += 1
    return _balls_on_polylines(rng, lines, radii, counts)


def vessel_tree(rng, n_balls, n_branches, half, r_root=1.5, r_min=0.3):
    """Random-walk branches; each new branch starts on an existing one."""
    lines, radii = [], []
    root = _random_walk(rng, np.array([0.0, 0.0, -0.8 * half]),
                        np.array([0.0, 0.0, 1.0]), 1.6 * half, half)
    lines.append(root)
    radii.append(r_root)
    gen = [0]
    while len(lines) < n_branches:
        parent = int(rng.integers(0, len(lines)))
        pts = lines[parent]
        start = pts[int(rng.integers(0, len(pts)))]
        g = gen[parent] + 1
        r = max(r_min, radii[parent] * 0.79)      # Murray-like taper
        length = max(4.0, half * rng.uniform(0.5, 1.2) * 0.85 ** g)
        lines.append(_random_walk(rng, start, rng.normal(size=3), length,
                                  half))
        radii.append(r)
        gen.append(g)
    w = np.array([len(p) * r for p, r in zip(lines, radii)], dtype=float)
    counts = np.floor(n_balls * w / w.sum()).astype(int)
    counts[: n_balls - counts.sum()] += 1
    return _balls_on_polylines(rng, lines, radii, counts)


@dataclass
class Problem:
    """One seeded BASELINE configuration."""

    name: str
    array: SensorArray
    frame_times: np.ndarray
    gt_frames: list                 # per frame (a0, p0, mu) float64 arrays
    cloud: DynamicCloud             # model parameters at iteration 0
    config: ReconConfig
    meta: dict = field(default_factory=dict)

    @property
    def n_frames(self) -> int:
        return len(self.frame_times)


CONFIG_SHAPES = {
    1: dict(B=4096, M=256, T=2048, F=1),
    2: dict(B=20000, M=512, T=4096, F=8),
    3: dict(B=200000, M=1024, T=4096, F=32),
    4: dict(B=1000000, M=2048, T=8192, F=16),
    5: dict(B=50000, M=512, T=4096, F=16),
}


def _motion(rng, mu, a0, axes, F, amp=0.08, period=8.0, drift=0.5):
    frames = []
    for k in range(F):
        s = 1.0 + amp * np.sin(2 * np.pi * k / period)
        d = drift * np.array([np.sin(2 * np.pi * k / period),
                              0.5 * np.sin(4 * np.pi * k / period), 0.0])
        frames.append((q32(a0 * s), None, q32(axes + s * (mu - axes) + d)))
    return frames


def make_problem(cfg_id: int, seed: int | None = None, scale: float = 1.0,
                 n_balls: int | None = None, n_sensors: int | None = None,
                 n_frames: int | None = None, n_samples: int | None = None,
                 basis: str = "polyfourier", n_basis: int | None = None
                 ) -> Problem:
    """Build BASELINE config `cfg_id` (1-5); sizes may be overridden (tests
    use reduced instances with the same distributions)."""
    shp = dict(CONFIG_SHAPES[cfg_id])
    if n_balls is not None:
        shp["B"] = n_balls
    elif scale != 1.0:
        shp["B"] = max(1, int(shp["B"] * scale))
    if n_sensors is not None:
        shp["M"] = n_sensors
    if n_frames is not None:
        shp["F"] = n_frames
    if n_samples is not None:
        shp["T"] = n_samples
    B, M, T, F = shp["B"], shp["M"], shp["T"], shp["F"]
    rng = np.random.default_rng(cfg_id if seed is None else seed)
    if cfg_id == 1:
        mu = q32(np.column_stack([rng.uniform(-10, 10, B),
                                  rng.uniform(-10, 10, B),
                                  rng.uniform(10, 30, B)]))
        p0 = q32(rng.uniform(0.1, 1.0, B))
        s_log = 0.3
        a0 = q32(np.clip(rng.lognormal(np.log(0.2) - 0.5 * s_log ** 2, s_log,
                                       B), 0.1, 0.4))
        mu_obs = q32(mu + rng.normal(0.0, 0.05, (B, 3)))
        side = int(round(np.sqrt(M)))
        pos = q32(planar_grid(side, 2.0)) if side * side == M else \
            q32(planar_grid(16, 2.0)[:M])
        array = SensorArray(pos, 1.5, 40.0, T, 0.0)
        cloud = DynamicCloud(p0, a0, mu, None, None, np.zeros((B, 5, 8)),
                             basis="polyfourier")
        cfg = ReconConfig(basis="polyfourier", n_basis=8)
        return Problem("config1", array, frame_times(1),
                       [(a0, p0, mu_obs)], cloud, cfg,
                       {"shape": shp, "seed": seed})
    half = {2: 15.0, 3: 20.0, 4: 30.0, 5: 15.0}[cfg_id]
    radius = {2: 40.0, 3: 60.0, 4: 60.0, 5: 40.0}[cfg_id]
    if cfg_id == 2:
        mu, a0, axes = tubes(rng, B, 12, 30.0, 0.3, 1.5, half)
    else:
        mu, a0, axes = vessel_tree(rng, B, 64, half)
    p0 = q32(rng.uniform(0.5, 1.0, B))
    a0 = q32(np.clip(a0, 0.1, None))
    mu = q32(mu)
    pos = q32(hemisphere(M, radius))
    array = SensorArray(pos, 1.5, 40.0, T, 0.0)
    gt = [(a_, p0, m_) for a_, _, m_ in _motion(rng, mu, a0, axes, F)]
    if basis == "gauss":
        # the reference's own default model: Gaussian basis on the default
        # grid (core.py:152-163, n_basis 65 by default, core.py:468)
        nb = 65 if n_basis is None else int(n_basis)
        th, sg = default_basis_grid(nb)
        omega = q32(rng.uniform(-0.01, 0.01, (B, 5, nb)))
        cloud = DynamicCloud(p0, a0, mu, np.tile(th, (B, 1)),
                             np.tile(sg, (B, 1)), omega)
        cfg = ReconConfig(n_basis=nb)
    else:
        omega = q32(rng.uniform(-0.01, 0.01, (B, 5, 8)))
        cloud = DynamicCloud(p0, a0, mu, None, None, omega,
                             basis="polyfourier")
        cfg = ReconConfig(basis="polyfourier", n_basis=8)
    return Problem(f"config{cfg_id}", array, frame_times(F), gt, cloud, cfg,
                   {"shape": shp, "seed": seed, "half": half,
                    "radius": radius})
