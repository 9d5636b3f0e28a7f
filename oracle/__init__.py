"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the 4D SlingBAG hot path.

A float64 restatement of the reference ``pacloud`` algorithm for the path
deform -> forward -> L2 loss -> adjoint -> deformation chain rule -> Adam /
floors, plus prune / split compaction.  It is the checker for the CUDA path
and the timed CPU baseline of ``bench.py``; nothing in
``paper_2412_03898_b200`` imports it (the product fails loudly without its
CUDA library instead of falling back here).

Pinning (see tests/test_oracle.py):
  * radiator kernels, deformation, chain rule, loss, Adam and prune are
    checked against golden vectors produced by the live reference
    (tests/golden/make_golden.py, run in the build container where
    /root/reference exists) and against the reference's own known-answer
    tests (test_radiator.py, test_deformation.py, test_reconstruction.py).
  * the poly+Fourier basis and the split/absolute-prune densify rule are
    NOT in the reference: they are builder-defined here
    and their parity is "unpinned by reference tests".
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libradiator_oracle.so"
_lib = None

N_CHANNELS = 5
COORD_MODES = ("multiplicative", "additive", "radial")
ADAM_BETA1, ADAM_BETA2, ADAM_EPS = 0.9, 0.999, 1e-8   # reconstruction.py:23-25


def build() -> Path:
    """Compile the C restatement (oracle/Makefile) if it is missing or stale."""
    src = _HERE / "radiator_oracle.c"
    if (not _LIB_PATH.exists()
            or _LIB_PATH.stat().st_mtime < src.stat().st_mtime):
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lp = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_forward_traces.argtypes = [
            dp, dp, dp, i64, dp, i64, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, i64, ctypes.c_double, ctypes.c_int, dp, lp,
            ctypes.c_int]
        lib.oracle_residual_state_grads.argtypes = [
            dp, dp, dp, i64, dp, i64, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, dp, i64, ctypes.c_double, ctypes.c_int, dp, lp,
            ctypes.c_int]
        lib.oracle_support_samples.argtypes = [
            dp, dp, i64, dp, i64, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, i64, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        lib.oracle_support_samples.restype = i64
        lib.oracle_backproject.argtypes = [
            dp, dp, i64, i64, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, i64, i64, i64, dp, ctypes.c_int]
        lib.oracle_voxelize.argtypes = [
            dp, dp, dp, i64, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, i64, i64, i64, ctypes.c_double,
            ctypes.c_int, dp, ctypes.c_int]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


# --------------------------------------------------------------------------
# simple containers (duck-compatible with the reference's types)
# --------------------------------------------------------------------------

@dataclass
class States:
    """Per-ball instantaneous attributes (deformation.py:31-54 CloudState)."""
    a0_t: np.ndarray
    p0_t: np.ndarray
    mu_t: np.ndarray

    def __len__(self):
        return self.a0_t.shape[0]


@dataclass
class Jacobian:
    """deformation.py:207-216 CloudStateGrad."""
    d_base: np.ndarray
    d_omega: np.ndarray
    d_theta: np.ndarray
    d_sigma: np.ndarray
    omega_row: np.ndarray
    shared_basis: bool


@dataclass
class Grads:
    """radiator.py:245-263 CloudGrads (parameter gradients)."""
    p0: np.ndarray
    a0: np.ndarray
    mu: np.ndarray
    theta: np.ndarray
    sigma: np.ndarray
    omega: np.ndarray

    def flat(self):
        return np.concatenate([self.p0.ravel(), self.a0.ravel(),
                               self.mu.ravel(), self.theta.ravel(),
                               self.sigma.ravel(), self.omega.ravel()])

    def add(self, o):
        for k in ("p0", "a0", "mu", "theta", "sigma", "omega"):
            setattr(self, k, getattr(self, k) + getattr(o, k))
        return self


# --------------------------------------------------------------------------
# radiator (C kernels) -- radiator.py:195-242
# --------------------------------------------------------------------------

def _array_fields(array):
    pos = np.ascontiguousarray(array.positions, dtype=np.float64)
    return (pos, float(array.sound_speed), float(array.t_start),
            1.0 / float(array.sample_rate), int(array.n_samples))


def forward_frame(states, array, support_sigmas=6.0, exact=False,
                  threads=0):
    """radiator.py:195-216; returns (M, T) float64 traces."""
    pos, v, t0, dt, T = _array_fields(array)
    M = pos.shape[0]
    out = np.zeros((M, T))
    B = len(states.a0_t)
    if B == 0:
        return out
    a0 = np.ascontiguousarray(states.a0_t, dtype=np.float64)
    if np.any(a0 <= 0):
        raise ValueError("all a0_t must be > 0 (clamp before the radiator)")
    p0 = np.ascontiguousarray(states.p0_t, dtype=np.float64)
    mu = np.ascontiguousarray(states.mu_t, dtype=np.float64)
    flag = np.zeros(1, dtype=np.int64)
    _load().oracle_forward_traces(
        _dp(mu), _dp(a0), _dp(p0), B, _dp(pos), M, v, t0, dt, T,
        float(support_sigmas), int(bool(exact)), _dp(out),
        flag.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(threads))
    if flag[0]:
        _raise_coincident(mu, pos)
    return out


def frame_state_grads(states, array, residual, support_sigmas=6.0,
                      exact=False, threads=0):
    """radiator.py:219-242; returns G (B, 5) in state order."""
    pos, v, t0, dt, T = _array_fields(array)
    M = pos.shape[0]
    residual = np.ascontiguousarray(residual, dtype=np.float64)
    if residual.shape != (M, T):
        raise ValueError(f"residual shape {residual.shape} does not match "
                         f"the array ({M}, {T})")
    B = len(states.a0_t)
    G = np.zeros((B, 5))
    if B == 0:
        return G
    a0 = np.ascontiguousarray(states.a0_t, dtype=np.float64)
    p0 = np.ascontiguousarray(states.p0_t, dtype=np.float64)
    mu = np.ascontiguousarray(states.mu_t, dtype=np.float64)
    flag = np.zeros(1, dtype=np.int64)
    _load().oracle_residual_state_grads(
        _dp(mu), _dp(a0), _dp(p0), B, _dp(pos), M, v, t0, dt, _dp(residual),
        T, float(support_sigmas), int(bool(exact)), _dp(G),
        flag.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(threads))
    if flag[0]:
        _raise_coincident(mu, pos)
    return G


def support_samples(states, array, support_sigmas=6.0, exact=False,
                    threads=0) -> int:
    """Exact sum over pairs of the in-support window length."""
    pos, v, t0, dt, T = _array_fields(array)
    a0 = np.ascontiguousarray(states.a0_t, dtype=np.float64)
    mu = np.ascontiguousarray(states.mu_t, dtype=np.float64)
    return int(_load().oracle_support_samples(
        _dp(mu), _dp(a0), len(a0), _dp(pos), pos.shape[0], v, t0, dt, T,
        float(support_sigmas), int(bool(exact)), int(threads)))


def _raise_coincident(mu, pos):
    """radiator.py:186-192 error message."""
    d = np.linalg.norm(mu[:, None, :] - pos[None, :, :], axis=2)
    b, m = np.unravel_index(np.argmin(d), d.shape)
    raise ValueError(f"ball {b} coincides with sensor {m} "
                     f"(distance {d[b, m]:.3g} mm)")


# --------------------------------------------------------------------------
# deformation -- deformation.py:87-99, 184-267 (Gaussian basis) and the
# builder-defined poly+Fourier basis (BASELINE configs 2-5; unpinned)
# --------------------------------------------------------------------------

def state_rows(coord_mode):
    """deformation.py:87-90: omega row that drives each state."""
    if coord_mode not in COORD_MODES:
        raise ValueError(f"coord_mode must be one of {COORD_MODES}")
    return np.array([0, 1, 2, 2, 2]) if coord_mode == "radial" \
        else np.arange(5)


def gauss_pieces(t, theta, sigma):
    """deformation.py:93-99: basis value and its theta / sigma partials."""
    u = (t - theta) / sigma
    val = np.exp(-0.5 * u * u)
    return val, val * u / sigma, val * u * u / sigma


def polyfourier_basis(t, n_harmonics=2):
    """Fixed basis [1, t, t^2, t^3, sin 2pi k t, cos 2pi k t (k=1..K)].

    Builder-defined (BASELINE config 2: "cubic polynomial in t plus 2
    Fourier terms"); period = the normalised clip [0, 1].  Unpinned.
    """
    t = float(t)
    vals = [1.0, t, t * t, t * t * t]
    for k in range(1, n_harmonics + 1):
        w = 2.0 * np.pi * k * t
        vals += [np.sin(w), np.cos(w)]
    return np.array(vals)


def _basis_table(cloud, t, basis):
    """phi (B, N) [shared] or (B, 5, N) [per-channel] plus partials."""
    if basis == "polyfourier":
        nb = cloud.omega.shape[-1]
        phi = np.broadcast_to(polyfourier_basis(t, (nb - 4) // 2),
                              (cloud.omega.shape[0], nb))
        z = np.zeros_like(phi)
        return phi, z, z
    return gauss_pieces(t, cloud.theta, cloud.sigma)


def _channel_sums(omega, phi):
    if phi.ndim == 2:
        return np.einsum("bcn,bn->bc", omega, phi)
    return np.sum(omega * phi, axis=2)


def cloud_states_at(cloud, t, coord_mode="multiplicative", a0_floor=None,
                    basis="gauss"):
    """deformation.py:184-204."""
    rows = state_rows(coord_mode)
    phi, _, _ = _basis_table(cloud, t, basis)
    H = _channel_sums(cloud.omega, phi)
    a0_t = cloud.a0 * (1.0 + H[:, 0])
    p0_t = cloud.p0 * (1.0 + H[:, 1])
    hmu = H[:, rows[2:]]
    mu_t = cloud.mu + hmu if coord_mode == "additive" \
        else cloud.mu * (1.0 + hmu)
    if a0_floor is not None:
        a0_t = np.maximum(a0_t, a0_floor)
    return States(a0_t, p0_t, np.ascontiguousarray(mu_t))


def cloud_state_grads(cloud, t, coord_mode="multiplicative", a0_floor=None,
                      basis="gauss"):
    """deformation.py:219-267 (materialised Jacobian bundle)."""
    rows = state_rows(coord_mode)
    phi, dth, dsg = _basis_table(cloud, t, basis)
    B, nb = cloud.omega.shape[0], cloud.omega.shape[-1]
    shared = phi.ndim == 2
    if shared:
        phi5 = np.broadcast_to(phi[:, None, :], (B, 5, nb))
        dth5 = np.broadcast_to(dth[:, None, :], (B, 5, nb))
        dsg5 = np.broadcast_to(dsg[:, None, :], (B, 5, nb))
    else:
        phi5, dth5, dsg5 = phi, dth, dsg
    H = np.sum(cloud.omega * phi5, axis=2)
    factor = np.column_stack([cloud.a0, cloud.p0, cloud.mu])
    if coord_mode == "additive":
        factor[:, 2:] = 1.0
        d_base = np.ones((B, 5))
        d_base[:, :2] = 1.0 + H[:, :2]
    else:
        d_base = 1.0 + H[:, rows]
    w_sel = cloud.omega[:, rows, :]
    d_omega = factor[:, :, None] * phi5[:, rows, :]
    d_theta = factor[:, :, None] * w_sel * dth5[:, rows, :]
    d_sigma = factor[:, :, None] * w_sel * dsg5[:, rows, :]
    if a0_floor is not None:
        hit = cloud.a0 * (1.0 + H[:, 0]) < a0_floor
        d_base[hit, 0] = 0.0
        d_omega[hit, 0, :] = 0.0
        d_theta[hit, 0, :] = 0.0
        d_sigma[hit, 0, :] = 0.0
    return Jacobian(d_base, np.ascontiguousarray(d_omega),
                    np.ascontiguousarray(d_theta),
                    np.ascontiguousarray(d_sigma), rows, shared)


def assemble_grads(G, jac: Jacobian, basis="gauss"):
    """radiator.py:278-294: chain rule of G (B,5) through the Jacobian."""
    B, _, nb = jac.d_omega.shape
    gb = G * jac.d_base
    c_om = G[:, :, None] * jac.d_omega
    c_th = G[:, :, None] * jac.d_theta
    c_sg = G[:, :, None] * jac.d_sigma
    g_om = np.zeros((B, 5, nb))
    np.add.at(g_om, (slice(None), jac.omega_row), c_om)
    if basis == "polyfourier":
        g_th = np.zeros((B, 0))
        g_sg = np.zeros((B, 0))
    elif jac.shared_basis:
        g_th = c_th.sum(axis=1)
        g_sg = c_sg.sum(axis=1)
    else:
        g_th = np.zeros((B, 5, nb))
        g_sg = np.zeros((B, 5, nb))
        np.add.at(g_th, (slice(None), jac.omega_row), c_th)
        np.add.at(g_sg, (slice(None), jac.omega_row), c_sg)
    return Grads(gb[:, 1].copy(), gb[:, 0].copy(), gb[:, 2:5].copy(), g_th,
                 g_sg, g_om)


# --------------------------------------------------------------------------
# loss and optimiser -- reconstruction.py:28-76, 153-157
# --------------------------------------------------------------------------

def l2_loss(predicted, observed):
    """reconstruction.py:28-35."""
    p = np.asarray(predicted, dtype=np.float64)
    o = np.asarray(observed, dtype=np.float64)
    if p.shape != o.shape:
        raise ValueError(f"shape mismatch: {p.shape} vs {o.shape}")
    d = p - o
    return 0.5 * float(np.sum(d * d))


def scheduled_lr(lr0, iteration, step_size, drop_rate):
    """reconstruction.py:38-41."""
    return lr0 * drop_rate ** (iteration // step_size)


@dataclass
class Moments:
    m: np.ndarray
    v: np.ndarray
    t: int = 0


def adam_step(param, grad, st: Moments, lr, group=""):
    """reconstruction.py:57-69 (in place)."""
    if not np.all(np.isfinite(grad)):
        raise ValueError(f"non-finite gradient in parameter group '{group}'")
    st.t += 1
    st.m *= ADAM_BETA1
    st.m += (1.0 - ADAM_BETA1) * grad
    st.v *= ADAM_BETA2
    st.v += (1.0 - ADAM_BETA2) * grad * grad
    mh = st.m / (1.0 - ADAM_BETA1 ** st.t)
    vh = st.v / (1.0 - ADAM_BETA2 ** st.t)
    param -= lr * mh / (np.sqrt(vh) + ADAM_EPS)


def sgd_step(param, grad, lr, group=""):
    """reconstruction.py:72-76."""
    if not np.all(np.isfinite(grad)):
        raise ValueError(f"non-finite gradient in parameter group '{group}'")
    param -= lr * grad


# --------------------------------------------------------------------------
# one dynamic iteration -- reconstruction.py:293-328
# --------------------------------------------------------------------------

GROUP_ORDER = ("pressure", "std", "coords", "deform")   # :320-327


def group_arrays(cloud, basis="gauss"):
    """Parameter arrays per optimiser group, in update order."""
    deform = {"omega": cloud.omega} if basis == "polyfourier" else \
        {"theta": cloud.theta, "sigma": cloud.sigma, "omega": cloud.omega}
    return {"pressure": {"p0": cloud.p0}, "std": {"a0": cloud.a0},
            "coords": {"mu": cloud.mu}, "deform": deform}


def iteration_grads(cloud, frame_times, observed_fmt, array, cfg,
                    basis="gauss", threads=0):
    """Loss and summed parameter gradients over the selected frames.

    observed_fmt: (F, M, T) observed traces of the selected frames.
    cfg: any object with coord_mode, a0_floor, support_sigmas, exact_forward.
    """
    loss = 0.0
    acc = None
    for k, t in enumerate(frame_times):
        st = cloud_states_at(cloud, float(t), cfg.coord_mode, cfg.a0_floor,
                             basis)
        jac = cloud_state_grads(cloud, float(t), cfg.coord_mode,
                                cfg.a0_floor, basis)
        pred = forward_frame(st, array, cfg.support_sigmas,
                             cfg.exact_forward, threads)
        r = pred - observed_fmt[k]
        loss += 0.5 * float(np.sum(r * r))
        G = frame_state_grads(st, array, r, cfg.support_sigmas,
                              cfg.exact_forward, threads)
        g = assemble_grads(G, jac, basis)
        acc = g if acc is None else acc.add(g)
    return loss, acc


def apply_step(cloud, grads: Grads, moments, lrs, cfg, basis="gauss"):
    """reconstruction.py:320-328: four Adam groups then the floors."""
    arrays = group_arrays(cloud, basis)
    for gname in GROUP_ORDER:
        for key, param in arrays[gname].items():
            adam_step(param, getattr(grads, key), moments[key], lrs[gname],
                      gname)
    np.maximum(cloud.p0, cfg.p0_floor, out=cloud.p0)
    np.maximum(cloud.a0, cfg.a0_floor, out=cloud.a0)
    if basis != "polyfourier":
        np.maximum(cloud.sigma, cfg.sigma_floor, out=cloud.sigma)


# --------------------------------------------------------------------------
# compaction -- reconstruction.py:95-100, 217-226 (prune, pinned) and the
# builder-defined split / absolute prune of BASELINE config 5 (unpinned)
# --------------------------------------------------------------------------

def prune_keep(p0, prune_threshold):
    """reconstruction.py:218-220: keep = p0 > thr * max(p0, initial=0)."""
    thr = prune_threshold * float(np.max(p0, initial=0.0))
    return p0 > thr


def compact(arr, keep):
    """reconstruction.py:95-100: stable boolean gather along axis 0."""
    return arr[keep]


def percentile_linear(x, q):
    """numpy percentile, method='linear' (numpy/lib/_function_base_impl)."""
    return float(np.percentile(x, q))


def densify_plan(p0, gp0, p0_min=0.01, q=90.0, max_balls=None):
    """Config-5 rule (builder-defined, unpinned).

    prune: p0 < p0_min (strict); split: |gp0| > P_q(|gp0|) (strict, numpy
    linear percentile over all balls) and not pruned.  New order is the
    survivors in parent order followed by one child per split survivor, in
    parent order.  Returns (keep mask, split mask, gather index of the new
    cloud, is_child flags).
    """
    g = np.abs(np.asarray(gp0, dtype=np.float64))
    keep = ~(np.asarray(p0) < p0_min)
    thr = percentile_linear(g, q) if g.size else 0.0
    split = (g > thr) & keep
    survivors = np.nonzero(keep)[0]
    children = np.nonzero(split)[0]
    if max_balls is not None:
        # cap: the first (max_balls - #survivors) split balls, parent order
        children = children[:max(0, int(max_balls) - len(survivors))]
        split = np.zeros_like(split)
        split[children] = True
    index = np.concatenate([survivors, children]).astype(np.int64)
    is_child = np.concatenate([np.zeros(len(survivors), bool),
                               np.ones(len(children), bool)])
    return keep, split, index, is_child


def apply_densify(params: dict, index, is_child, split, keep,
                  child_shift=0.5, halve_pressure=False):
    """Gather survivors + children (clones of their parents); with
    `halve_pressure` halve p0 of split parents and children; shift each
    child's centre by +child_shift*a0 along x (builder-defined).
    `params` maps name -> (B, ...) array; Adam moments are gathered with the
    same index and zeroed for children by the caller."""
    out = {k: np.array(v[index]) for k, v in params.items()}
    if halve_pressure:
        halve = split[index]
        out["p0"] = np.where(halve, 0.5 * out["p0"], out["p0"])
    if "mu" in out:
        shift = np.where(is_child, child_shift * out["a0"], 0.0)
        out["mu"][:, 0] = out["mu"][:, 0] + shift
    return out


# --------------------------------------------------------------------------
# static stage -- reconstruction.py:160-231
# --------------------------------------------------------------------------

def lattice_1d(lo, hi, pitch):
    """geometry.py:121-126."""
    n = max(1, int(np.floor((hi - lo) / pitch + 1e-12)))
    return 0.5 * (lo + hi) - 0.5 * (n - 1) * pitch + pitch * np.arange(n)


def box_lattice(lo, hi, pitch):
    """geometry.py:129-132 (x slowest)."""
    ax = [lattice_1d(lo[k], hi[k], pitch) for k in range(3)]
    return np.stack(np.meshgrid(*ax, indexing="ij"), -1).reshape(-1, 3)


def static_reconstruct(observed, array, cfg, roi_lo, roi_hi, losses=None,
                       threads=0):
    """Lattice init, then per iteration forward -> loss -> adjoint -> Adam
    (pressure, std, coords) -> floors -> prune every prune_every.
    Returns (p0, a0, mu) float64 arrays."""
    observed = np.asarray(observed, dtype=np.float64)
    mu = box_lattice(roi_lo, roi_hi, cfg.init_pitch)
    a0 = np.full(len(mu), cfg.init_pitch / 2.0)
    peak = float(np.max(np.abs(observed))) if observed.size else 0.0
    p0 = np.full(len(mu), cfg.init_p0_scale * peak)
    mom = {k: Moments(np.zeros_like(v), np.zeros_like(v))
           for k, v in (("p0", p0), ("a0", a0), ("mu", mu))}
    for it in range(cfg.static_iters):
        lr = {g: scheduled_lr(getattr(cfg, "lr_" + g), it, cfg.step_size,
                              cfg.drop_rate)
              for g in ("pressure", "std", "coords")}
        st = States(a0, p0, mu)
        r = forward_frame(st, array, cfg.support_sigmas, cfg.exact_forward,
                          threads) - observed
        loss = 0.5 * float(np.sum(r * r))
        if not np.isfinite(loss):
            raise RuntimeError(f"non-finite loss at iteration {it}")
        if losses is not None:
            losses.append(loss)
        G = frame_state_grads(st, array, r, cfg.support_sigmas,
                              cfg.exact_forward, threads)
        step = adam_step if cfg.optimizer == "adam" else None
        for key, arr, g, grp in (("p0", p0, G[:, 1], "pressure"),
                                 ("a0", a0, G[:, 0], "std"),
                                 ("mu", mu, G[:, 2:5], "coords")):
            if step is not None:
                step(arr, g, mom[key], lr[grp], grp)
            else:
                sgd_step(arr, g, lr[grp], grp)
        np.maximum(p0, cfg.p0_floor, out=p0)
        np.maximum(a0, cfg.a0_floor, out=a0)
        if (it + 1) % cfg.prune_every == 0:
            keep = prune_keep(p0, cfg.prune_threshold)
            if not keep.any():
                raise RuntimeError("all balls pruned")
            if not keep.all():
                p0, a0, mu = p0[keep], a0[keep], mu[keep]
                for m in mom.values():
                    m.m, m.v = m.m[keep], m.v[keep]
    return p0, a0, mu


# ---------------------------------------------------------------- evaluation

def voxelize(mu, a0, p0, origin, spacing, dims, support_sigmas=6.0,
             exact=False, threads=0) -> np.ndarray:
    """evaluation.py:46-93: (nx, ny, nz) float64 Gaussian field at voxel
    centres origin + i * spacing (C restatement of _splat_balls)."""
    mu = np.ascontiguousarray(mu, dtype=np.float64).reshape(-1, 3)
    a0 = np.ascontiguousarray(a0, dtype=np.float64).ravel()
    p0 = np.ascontiguousarray(p0, dtype=np.float64).ravel()
    if len(a0) and np.any(a0 <= 0):
        raise ValueError("all a0_t must be > 0")
    dims = tuple(int(d) for d in dims)
    out = np.zeros(dims)
    o = np.asarray(origin, dtype=np.float64)
    _load().oracle_voxelize(_dp(mu), _dp(a0), _dp(p0), len(a0), o[0], o[1],
                            o[2], float(spacing), dims[0], dims[1], dims[2],
                            float(support_sigmas), int(bool(exact)), _dp(out),
                            int(threads))
    return out


def ssim(a, b, data_range=1.0, window=11, sigma=1.5, k1=0.01, k2=0.03):
    """evaluation.py:142-184: mean SSIM over fully contained Gaussian
    windows (numpy, float64)."""
    from numpy.lib.stride_tricks import sliding_window_view
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    r = np.arange(window, dtype=np.float64) - (window - 1) / 2.0
    g = np.exp(-0.5 * (r / sigma) ** 2)
    w = np.outer(g, g)
    w /= w.sum()

    def filt(img):
        return np.einsum("ijkl,kl->ij", sliding_window_view(img, w.shape), w)
    c1, c2 = (k1 * data_range) ** 2, (k2 * data_range) ** 2
    ma, mb = filt(a), filt(b)
    va, vb = filt(a * a) - ma * ma, filt(b * b) - mb * mb
    cov = filt(a * b) - ma * mb
    return float(np.mean((2 * ma * mb + c1) * (2 * cov + c2) /
                         ((ma * ma + mb * mb + c1) * (va + vb + c2))))


def ubp_reconstruct(traces, array, origin, spacing, dims, threads=0):
    """reconstruction.py:380-417 (window check omitted): numpy filter
    b = 2 p - 2 t dp/dt (np.gradient), C restatement of _backproject.
    Returns (nx, ny, nz) float64."""
    pos, v, t0, dt, T = _array_fields(array)
    traces = np.ascontiguousarray(traces, dtype=np.float64)
    times = array.t_start + np.arange(array.n_samples) / array.sample_rate
    filt = np.ascontiguousarray(
        2.0 * traces - 2.0 * times[None, :] * np.gradient(traces, dt, axis=1))
    dims = tuple(int(d) for d in dims)
    out = np.zeros(dims)
    o = np.asarray(origin, dtype=np.float64)
    _load().oracle_backproject(_dp(filt), _dp(pos), pos.shape[0], T, v, t0,
                               dt, o[0], o[1], o[2], float(spacing), dims[0],
                               dims[1], dims[2], _dp(out), int(threads))
    return out
