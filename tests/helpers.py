"""Shared test utilities (tolerances are BASELINE.json's)."""

import numpy as np

SIGNAL_TOL = 1e-5   # simulated signals, relative L2 (BASELINE north_star)
GRAD_TOL = 1e-4     # gradients, relative L2


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def small_array(golden, cls):
    c = golden["small_cfg"]
    return cls(golden["small_pos"], float(c[0]), float(c[1]), int(c[2]),
               float(c[3]))


def planar_array(golden, cls):
    return cls(golden["planar_pos"], 1.5, 40.0, 2048, 0.0)


def rel_err(analytic, numeric, scale=None, floor_rel=1e-9):
    """Elementwise relative error with a zero floor (reference oracles.py)."""
    a = np.asarray(analytic, dtype=np.float64)
    n = np.asarray(numeric, dtype=np.float64)
    if scale is None:
        scale = max(np.max(np.abs(a)), np.max(np.abs(n)), 1.0)
    denom = np.maximum(np.maximum(np.abs(a), np.abs(n)), floor_rel * scale)
    return np.abs(a - n) / denom


def fd_gradient(f, x, step):
    x = np.asarray(x, dtype=np.float64)
    g = np.zeros_like(x)
    for i in range(x.size):
        h = step * max(1.0, abs(x.flat[i]))
        xp = x.copy()
        xp.flat[i] += h
        xm = x.copy()
        xm.flat[i] -= h
        g.flat[i] = (f(xp) - f(xm)) / (2.0 * h)
    return g
