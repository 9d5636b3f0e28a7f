"""Drop-in deformation on the B200.

Mirrors pkg/src/pacloud/deformation.py -- ``cloud_states_at`` (:184-204) and
``cloud_state_grads`` (:219-267), same signatures -- plus a batched-over-
frames device layer (``DeviceCloud``, ``deform_states_device``,
``deform_backward_device``) used by the fused engine.  Arithmetic runs in
libpacloud_b200.so (pc_deform_states / pc_deform_jacobian /
pc_deform_backward).

States come back with a0_t / p0_t in float32 (the radiator's arithmetic
type) and mu_t in float64; ω = 0 reproduces float32-representable baselines
bit-exactly, as deformation.py:119-120 requires.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .core import COORD_MODES, CloudState, CloudStateGrad
from .radiator import _device, _is_torch, to_device


def omega_rows(coord_mode: str) -> np.ndarray:
    """deformation.py:87-90."""
    if coord_mode == "radial":
        return np.array([0, 1, 2, 2, 2])
    return np.arange(5)


def _basis_of(cloud) -> str:
    return getattr(cloud, "basis", "gauss")


class DeviceCloud:
    """Device f64 views of a DynamicCloud's parameters + its pc_cloud_t.

    `tensors` may alias slices of the engine's flat parameter buffer.
    """

    def __init__(self, p0, a0, mu, theta, sigma, omega, basis="gauss"):
        _lib.load_library()
        self.basis = basis
        self.p0, self.a0, self.mu = p0, a0, mu
        self.theta, self.sigma, self.omega = theta, sigma, omega
        self.B = int(p0.shape[0])
        self.N = int(omega.shape[-1])
        self.per_channel = basis == "gauss" and theta is not None \
            and theta.dim() == 3
        self.struct = _lib.PcCloud(
            _lib.ptr(p0), _lib.ptr(a0), _lib.ptr(mu),
            _lib.ptr(theta) if basis == "gauss" else None,
            _lib.ptr(sigma) if basis == "gauss" else None,
            _lib.ptr(omega), self.B, self.N, int(self.per_channel),
            _lib.PC_BASIS[basis], 0)

    @classmethod
    def from_cloud(cls, cloud) -> "DeviceCloud":
        basis = _basis_of(cloud)
        f = lambda x: to_device(x, torch.float64)   # noqa: E731
        th = f(cloud.theta) if basis == "gauss" else None
        sg = f(cloud.sigma) if basis == "gauss" else None
        return cls(f(cloud.p0), f(cloud.a0), f(cloud.mu), th, sg,
                   f(cloud.omega), basis)


def deform_states_device(dcloud: DeviceCloud, t_frames, coord_mode,
                         a0_floor, mu_t=None, a0_t=None, p0_t=None, H=None):
    """pc_deform_states for all frames: mu_t (F,B,3) f64, a0_t/p0_t (F,B)
    f32, H (F,B,5) f32 channel sums."""
    lib = _lib.load_library()
    F, B = int(t_frames.shape[0]), dcloud.B
    dev = t_frames.device
    if mu_t is None:
        mu_t = torch.empty((F, B, 3), dtype=torch.float64, device=dev)
    if a0_t is None:
        a0_t = torch.empty((F, B), dtype=torch.float32, device=dev)
    if p0_t is None:
        p0_t = torch.empty((F, B), dtype=torch.float32, device=dev)
    if H is None:
        H = torch.empty((F, B, 5), dtype=torch.float32, device=dev)
    floor = math.nan if a0_floor is None else float(a0_floor)
    _lib.check(lib.pc_deform_states(
        ctypes.byref(dcloud.struct), _lib.ptr(t_frames), F,
        _lib.PC_COORD[coord_mode], floor, _lib.ptr(mu_t), _lib.ptr(a0_t),
        _lib.ptr(p0_t), _lib.ptr(H), _lib.stream()), "pc_deform_states")
    return mu_t, a0_t, p0_t, H


def deform_backward_device(dcloud: DeviceCloud, t_frames, coord_mode,
                           a0_floor, G, H, grads):
    """pc_deform_backward: `grads` maps p0/a0/mu/theta/sigma/omega to f32
    device tensors shaped like the cloud (overwritten)."""
    lib = _lib.load_library()
    floor = math.nan if a0_floor is None else float(a0_floor)
    gs = _lib.PcCloudGrads(
        _lib.ptr(grads["p0"]), _lib.ptr(grads["a0"]), _lib.ptr(grads["mu"]),
        _lib.ptr(grads.get("theta")), _lib.ptr(grads.get("sigma")),
        _lib.ptr(grads["omega"]))
    _lib.check(lib.pc_deform_backward(
        ctypes.byref(dcloud.struct), _lib.ptr(t_frames),
        int(t_frames.shape[0]), _lib.PC_COORD[coord_mode], floor,
        _lib.ptr(G), _lib.ptr(H), ctypes.byref(gs), _lib.stream()),
        "pc_deform_backward")


def _check_mode(coord_mode):
    if coord_mode not in COORD_MODES:
        raise ValueError(f"coord_mode must be one of {COORD_MODES}")


def cloud_states_at(cloud, t: float, coord_mode: str = "multiplicative",
                    a0_floor: float | None = None) -> CloudState:
    """Vectorised ball_state_at over a DynamicCloud (deformation.py:184)."""
    _check_mode(coord_mode)
    torch_io = _is_torch(cloud.p0, cloud.omega)
    dc = DeviceCloud.from_cloud(cloud)
    tf = torch.tensor([float(t)], dtype=torch.float64, device=_device())
    if dc.B == 0:
        z = torch.zeros(0, dtype=torch.float64, device=_device())
        st = (z, z.clone(), torch.zeros((0, 3), dtype=torch.float64,
                                         device=_device()))
    else:
        # float64 a0_t / p0_t like the reference's CloudState (the engine's
        # radiator path keeps its own float32 copies)
        lib = _lib.load_library()
        f64 = dict(dtype=torch.float64, device=_device())
        mu_t = torch.empty((1, dc.B, 3), **f64)
        a0_t = torch.empty((1, dc.B), **f64)
        p0_t = torch.empty((1, dc.B), **f64)
        floor = math.nan if a0_floor is None else float(a0_floor)
        _lib.check(lib.pc_deform_states_f64(
            ctypes.byref(dc.struct), _lib.ptr(tf), 1,
            _lib.PC_COORD[coord_mode], floor, _lib.ptr(mu_t), _lib.ptr(a0_t),
            _lib.ptr(p0_t), _lib.stream()), "pc_deform_states_f64")
        st = (a0_t[0], p0_t[0], mu_t[0])
    if not torch_io:
        st = tuple(x.cpu().numpy() for x in st)
    return CloudState(*st)


def cloud_state_grads(cloud, t: float, coord_mode: str = "multiplicative",
                      a0_floor: float | None = None) -> CloudStateGrad:
    """Vectorised ball_state_grad over a DynamicCloud (deformation.py:219)."""
    _check_mode(coord_mode)
    lib = _lib.load_library()
    torch_io = _is_torch(cloud.p0, cloud.omega)
    dc = DeviceCloud.from_cloud(cloud)
    B, N = dc.B, dc.N
    f64 = dict(dtype=torch.float64, device=_device())
    d_base = torch.zeros((B, 5), **f64)
    d_om = torch.zeros((B, 5, N), **f64)
    gauss = dc.basis == "gauss"
    d_th = torch.zeros((B, 5, N), **f64) if gauss else torch.zeros((B, 0), **f64)
    d_sg = torch.zeros((B, 5, N), **f64) if gauss else torch.zeros((B, 0), **f64)
    if B:
        floor = math.nan if a0_floor is None else float(a0_floor)
        _lib.check(lib.pc_deform_jacobian(
            ctypes.byref(dc.struct), float(t), _lib.PC_COORD[coord_mode],
            floor, _lib.ptr(d_base), _lib.ptr(d_om),
            _lib.ptr(d_th) if gauss else None,
            _lib.ptr(d_sg) if gauss else None, _lib.stream()),
            "pc_deform_jacobian")
    out = [d_base, d_om, d_th, d_sg]
    if not torch_io:
        out = [x.cpu().numpy() for x in out]
    shared = (not gauss) or not dc.per_channel
    return CloudStateGrad(*out, omega_rows(coord_mode), shared)


# ---------------------------------------------------------------- single ball

def eval_basis(t, theta, sigma):
    """deformation.py:57-70: exp(-(t - theta)^2 / (2 sigma^2)), broadcasting
    (pc_eval_basis, fp64 on the device)."""
    theta = np.asarray(theta, dtype=np.float64)
    sigma = np.asarray(sigma, dtype=np.float64)
    if np.any(sigma <= 0):
        raise ValueError("basis width sigma must be > 0")
    lib = _lib.load_library()
    arrs = np.broadcast_arrays(np.asarray(t, dtype=np.float64), theta, sigma)
    shape = arrs[0].shape
    dev = [torch.as_tensor(np.ascontiguousarray(x).reshape(-1),
                           device=_device()) for x in arrs]
    out = torch.empty(dev[0].numel(), dtype=torch.float64, device=_device())
    _lib.check(lib.pc_eval_basis(*[_lib.ptr(x) for x in dev], out.numel(),
                                 _lib.ptr(out), _lib.stream()),
               "pc_eval_basis")
    res = out.cpu().numpy().reshape(shape)
    return float(res) if res.ndim == 0 else res


def eval_H(t: float, omega, theta, sigma) -> float:
    """deformation.py:73-84: weighted Gaussian-basis sum; zero weights give
    exactly 0 (pc_eval_h, fp64 on the device)."""
    omega = np.asarray(omega, dtype=np.float64)
    theta = np.asarray(theta, dtype=np.float64)
    sigma = np.asarray(sigma, dtype=np.float64)
    if not (omega.shape == theta.shape == sigma.shape) or omega.ndim != 1:
        raise ValueError(
            f"omega, theta, sigma must be 1-d with equal lengths, got "
            f"{omega.shape}, {theta.shape}, {sigma.shape}")
    if not np.any(omega):
        return 0.0
    if np.any(sigma <= 0):
        raise ValueError("basis width sigma must be > 0")
    lib = _lib.load_library()
    dev = [torch.as_tensor(x, device=_device()) for x in (omega, theta, sigma)]
    out = torch.empty(1, dtype=torch.float64, device=_device())
    _lib.check(lib.pc_eval_h(float(t), *[_lib.ptr(x) for x in dev],
                             len(omega), _lib.ptr(out), _lib.stream()),
               "pc_eval_h")
    return float(out.item())


def _one_ball_cloud(ball, deform):
    """A one-ball Gaussian-basis DeviceCloud (shared (1,N) or per-channel
    (1,5,N) theta/sigma) for the single-ball drop-ins."""
    f = lambda x: torch.as_tensor(np.asarray(x, dtype=np.float64)[None],  # noqa: E731
                                  device=_device()).contiguous()
    return DeviceCloud(f(ball.p0), f(ball.a0), f(ball.mu), f(deform.theta),
                       f(deform.sigma), f(deform.omega), "gauss")


def ball_state_at(ball, deform, t: float, coord_mode: str = "multiplicative",
                  a0_floor: float | None = None):
    """deformation.py:102-130: one ball at normalized time t (the batched
    kernel on a one-ball cloud; zero weights reproduce the baseline
    bit-exactly)."""
    from .core import BallStateAtT
    _check_mode(coord_mode)
    lib = _lib.load_library()
    dc = _one_ball_cloud(ball, deform)
    f64 = dict(dtype=torch.float64, device=_device())
    tf = torch.tensor([float(t)], **f64)
    mu_t = torch.empty((1, 1, 3), **f64)
    a0_t = torch.empty((1, 1), **f64)
    p0_t = torch.empty((1, 1), **f64)
    floor = math.nan if a0_floor is None else float(a0_floor)
    _lib.check(lib.pc_deform_states_f64(
        ctypes.byref(dc.struct), _lib.ptr(tf), 1, _lib.PC_COORD[coord_mode],
        floor, _lib.ptr(mu_t), _lib.ptr(a0_t), _lib.ptr(p0_t), _lib.stream()),
        "pc_deform_states_f64")
    return BallStateAtT(float(a0_t.item()), float(p0_t.item()),
                        mu_t[0, 0].cpu().numpy())


class BallStateGrad:
    """deformation.py:133-150: partials of one ball's state (rows in state
    order a0_t, p0_t, mu_x, mu_y, mu_z)."""

    def __init__(self, d_base, d_omega, d_theta, d_sigma, omega_row,
                 shared_basis):
        self.d_base = d_base
        self.d_omega = d_omega
        self.d_theta = d_theta
        self.d_sigma = d_sigma
        self.omega_row = omega_row
        self.shared_basis = shared_basis


def ball_state_grad(ball, deform, t: float,
                    coord_mode: str = "multiplicative") -> BallStateGrad:
    """deformation.py:153-181: exact partials of ball_state_at (no floor;
    pc_deform_jacobian on a one-ball cloud)."""
    _check_mode(coord_mode)
    lib = _lib.load_library()
    dc = _one_ball_cloud(ball, deform)
    N = dc.N
    f64 = dict(dtype=torch.float64, device=_device())
    d_base = torch.zeros((1, 5), **f64)
    d_om = torch.zeros((1, 5, N), **f64)
    d_th = torch.zeros((1, 5, N), **f64)
    d_sg = torch.zeros((1, 5, N), **f64)
    _lib.check(lib.pc_deform_jacobian(
        ctypes.byref(dc.struct), float(t), _lib.PC_COORD[coord_mode],
        math.nan, _lib.ptr(d_base), _lib.ptr(d_om), _lib.ptr(d_th),
        _lib.ptr(d_sg), _lib.stream()), "pc_deform_jacobian")
    return BallStateGrad(d_base[0].cpu().numpy(), d_om[0].cpu().numpy(),
                         d_th[0].cpu().numpy(), d_sg[0].cpu().numpy(),
                         omega_rows(coord_mode), bool(deform.theta.ndim == 1))
