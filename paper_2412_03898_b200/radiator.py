"""Drop-in radiator: forward model and adjoint on the B200.

Mirrors pkg/src/pacloud/radiator.py -- ``forward_frame`` (:195-216),
``frame_state_grads`` (:219-242), ``accumulate_frame_grads`` (:266-294) and
``CloudGrads`` (:245-263) -- with the same signatures, return shapes and
exceptions.  NumPy inputs return float64 NumPy outputs (host copies in and
out); torch CUDA inputs stay on the device.  All arithmetic runs in
libpacloud_b200.so (pc_forward_traces / pc_residual_state_grads /
pc_assemble_grads); there is no CPU path.

``DeviceArray`` and the ``*_device`` functions are the zero-copy, batched-
over-frames layer the fused engine uses.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .core import BallStateAtT, CloudGrads, CloudState

DEFAULT_SUPPORT_SIGMAS = 6.0


def _device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` (copies NumPy / host inputs)."""
    if isinstance(x, torch.Tensor):
        dev = x.device if x.is_cuda else _device()
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype,
                           device=_device()).contiguous()


def _is_torch(*xs) -> bool:
    return any(isinstance(x, torch.Tensor) for x in xs)


def sensor_cluster_order(pos: np.ndarray, bits: int = 10) -> np.ndarray:
    """Z-order of the sensors: consecutive 8-sensor slots of the forward
    kernel are spatial neighbours, so their arrival windows overlap."""
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
    if len(pos) == 0:
        return np.zeros(0, dtype=np.int32)
    lo = pos.min(axis=0)
    span = np.maximum(pos.max(axis=0) - lo, 1e-12)
    q = np.minimum(((pos - lo) / span * (1 << bits)).astype(np.int64),
                   (1 << bits) - 1)
    code = np.zeros(len(pos), dtype=np.int64)
    for bit in range(bits):
        for ax in range(3):
            code |= ((q[:, ax] >> bit) & 1) << (3 * bit + ax)
    return np.argsort(code, kind="stable").astype(np.int32)


class DeviceArray:
    """A SensorArray resident on the device plus its pc_array_t."""

    def __init__(self, array, support_sigmas=DEFAULT_SUPPORT_SIGMAS,
                 exact=False, positions=None, sensor_offset=0):
        _lib.load_library()
        self.array = array
        self.positions = to_device(
            array.positions if positions is None else positions,
            torch.float64)
        self.M = int(self.positions.shape[0])
        self.T = int(array.n_samples)
        self.v = float(array.sound_speed)
        self.t0 = float(array.t_start)
        self.dt = 1.0 / float(array.sample_rate)
        self.support = float(support_sigmas)
        self.exact = bool(exact)
        n_total = int(np.shape(array.positions)[0])
        self.order = torch.as_tensor(
            sensor_cluster_order(self.positions.double().cpu().numpy()),
            dtype=torch.int32, device=self.positions.device)
        self.struct = _lib.PcArray(
            self.positions.data_ptr(), self.M, self.T, self.v, self.t0,
            self.dt, self.support, int(self.exact), int(sensor_offset),
            self.order.data_ptr(), n_total, 0)
        self.sensor_offset = int(sensor_offset)
        self.n_sensors_total = n_total

    def variant(self) -> int:
        """pc_forward_variant: 0 register-run forward, 1 legacy shared-memory
        trace forward, 2 register-run forward with TMA-staged ball tiles."""
        lib = _lib.load_library(require_cuda=False)
        return int(lib.pc_forward_variant(ctypes.byref(self.struct)))

    def plan(self, n_balls: int, n_frames: int) -> dict:
        """pc_forward_plan: time segment, segments, ball chunks, launches."""
        lib = _lib.load_library(require_cuda=False)
        out = (ctypes.c_int32 * 4)()
        _lib.check(lib.pc_forward_plan(int(n_balls), int(n_frames),
                                       ctypes.byref(self.struct), out),
                   "pc_forward_plan")
        return {"tseg": out[0], "nseg": out[1], "nchunk": out[2],
                "launches": out[3]}

    def workspace_bytes(self, n_balls: int, n_frames: int) -> int:
        lib = _lib.load_library()
        return int(lib.pc_forward_workspace_bytes(
            int(n_balls), int(n_frames), ctypes.byref(self.struct)))


_DARR_CACHE: "OrderedDict" = None


def cached_device_array(array, support_sigmas=DEFAULT_SUPPORT_SIGMAS,
                        exact=False) -> DeviceArray:
    """DeviceArray of a host SensorArray, reused across the per-frame
    drop-in calls (a patched reference loop calls forward_frame and
    accumulate_frame_grads once per frame with the same array): keyed by
    the array's scalars and a digest of its positions, 8 entries, LRU.
    Device-tensor positions are not cached."""
    global _DARR_CACHE
    from collections import OrderedDict
    import hashlib
    pos = array.positions
    if isinstance(pos, torch.Tensor):
        return DeviceArray(array, support_sigmas, exact)
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    key = (hashlib.blake2b(pos.tobytes(), digest_size=16).digest(), pos.shape,
           float(array.sound_speed), float(array.sample_rate),
           int(array.n_samples), float(array.t_start), float(support_sigmas),
           bool(exact), torch.cuda.current_device())
    if _DARR_CACHE is None:
        _DARR_CACHE = OrderedDict()
    d = _DARR_CACHE.get(key)
    if d is None:
        d = DeviceArray(array, support_sigmas, exact)
        _DARR_CACHE[key] = d
        if len(_DARR_CACHE) > 8:
            _DARR_CACHE.popitem(last=False)
    else:
        _DARR_CACHE.move_to_end(key)
    return d


def forward_device(darr: DeviceArray, mu_t, a0_t, p0_t, observed=None,
                   out=None, loss=None, coincident=None, workspace=None):
    """pc_forward_traces on device tensors.

    mu_t (F,B,3) f64, a0_t/p0_t (F,B) f32, observed (F,M,T) f32 or None.
    Returns (out, loss, coincident): out (F,M,T) f32 = predicted traces, or
    the residual predicted - observed when `observed` is given; loss (F,)
    f64 per frame (only with observed).
    """
    lib = _lib.load_library()
    F, B = int(a0_t.shape[0]), int(a0_t.shape[1])
    dev = a0_t.device
    if out is None:
        out = torch.empty((F, darr.M, darr.T), dtype=torch.float32,
                          device=dev)
    if observed is not None and loss is None:
        loss = torch.empty(F, dtype=torch.float64, device=dev)
    if coincident is None:
        coincident = torch.full((1,), _lib.INT64_MAX, dtype=torch.int64,
                                device=dev)
    need = darr.workspace_bytes(max(B, 1), F)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    _lib.check(lib.pc_forward_traces(
        _lib.ptr(mu_t), _lib.ptr(a0_t), _lib.ptr(p0_t), B, F,
        ctypes.byref(darr.struct), _lib.ptr(observed), _lib.ptr(out),
        _lib.ptr(loss) if observed is not None else None,
        _lib.ptr(coincident), _lib.ptr(workspace), workspace.numel(),
        _lib.stream()), "pc_forward_traces")
    return out, loss, coincident


def residual_loss_device(predicted, observed, out=None, loss=None,
                         partial=None):
    """pc_residual_loss: out = predicted - observed (in place when out is
    predicted), loss (F,) f64 = 0.5 * sum r^2 per frame."""
    lib = _lib.load_library()
    F, M, T = (int(x) for x in predicted.shape)
    dev = predicted.device
    if out is None:
        out = predicted
    if loss is None:
        loss = torch.empty(F, dtype=torch.float64, device=dev)
    if partial is None or partial.numel() < F * M:
        partial = torch.empty(F * M, dtype=torch.float64, device=dev)
    _lib.check(lib.pc_residual_loss(
        _lib.ptr(predicted), _lib.ptr(observed), _lib.ptr(out),
        _lib.ptr(partial), _lib.ptr(loss), F, M, T, _lib.stream()),
        "pc_residual_loss")
    return out, loss


def state_grads_device(darr: DeviceArray, mu_t, a0_t, p0_t, residual,
                       G=None, coincident=None):
    """pc_residual_state_grads: G (F,B,5) f32 from residual (F,M,T)."""
    lib = _lib.load_library()
    F, B = int(a0_t.shape[0]), int(a0_t.shape[1])
    dev = a0_t.device
    if G is None:
        G = torch.empty((F, B, 5), dtype=torch.float32, device=dev)
    if coincident is None:
        coincident = torch.full((1,), _lib.INT64_MAX, dtype=torch.int64,
                                device=dev)
    _lib.check(lib.pc_residual_state_grads(
        _lib.ptr(mu_t), _lib.ptr(a0_t), _lib.ptr(p0_t), B, F,
        ctypes.byref(darr.struct), _lib.ptr(residual), _lib.ptr(G),
        _lib.ptr(coincident), _lib.stream()), "pc_residual_state_grads")
    return G, coincident


def coincident_pair(mu, positions, chunk: int = 1 << 16):
    """radiator.py:186-192 _raise_coincident's pair: the first (ball, sensor)
    of the smallest distance |mu_b - s_m| in C order (numpy argmin), and
    that distance.  Computed on the device in ball chunks (fp64)."""
    mu = to_device(mu, torch.float64).reshape(-1, 3)
    pos = to_device(positions, torch.float64).reshape(-1, 3)
    best, bb, mm = math.inf, 0, 0
    for b0 in range(0, mu.shape[0], chunk):
        d = torch.sqrt(((mu[b0:b0 + chunk, None, :] - pos[None, :, :]) ** 2)
                       .sum(dim=2))
        k = int(torch.argmin(d).item())
        b, m = divmod(k, pos.shape[0])
        v = float(d[b, m].item())
        if v < best:
            best, bb, mm = v, b0 + b, m
    return bb, mm, best


def raise_if_coincident(coincident, mu_t, positions):
    """radiator.py:186-192: if the device coincidence word is set, raise the
    reference's ValueError naming the closest (ball, sensor) pair of the
    frame (mu_t: that frame's centres, positions: the whole array)."""
    c = int(coincident.item()) if isinstance(coincident, torch.Tensor) \
        else int(coincident)
    if c == _lib.INT64_MAX:
        return
    b, m, d = coincident_pair(mu_t, positions)
    raise ValueError(f"ball {b} coincides with sensor {m} "
                     f"(distance {d:.3g} mm)")


def compute_time_window(array, roi, margin_a0: float):
    """radiator.py:297-322: (t_start, n_samples) covering time of flight to
    the nearest / farthest ROI points (circumscribed about the origin),
    padded by 6 margin_a0 on each side, count rounded up."""
    if margin_a0 < 0:
        raise ValueError("margin_a0 must be >= 0")
    norms = np.linalg.norm(np.asarray(array.positions, float), axis=1)
    r_near, r_far = float(norms.min()), float(norms.max())
    r_roi = roi.circumradius()
    if r_roi >= r_near:
        raise ValueError(
            f"roi circumscribed radius {r_roi:.3f} mm reaches the sensor "
            f"sphere (nearest sensor at {r_near:.3f} mm)")
    pad = 6.0 * margin_a0
    t_lo = max(0.0, (r_near - r_roi - pad) / array.sound_speed)
    t_hi = (r_far + r_roi + pad) / array.sound_speed
    span = max(0.0, (t_hi - t_lo) * array.sample_rate - 1e-9)
    return t_lo, int(np.ceil(span)) + 1


# ---------------------------------------------------------------- drop-ins

def _eval_pressure(R, t, p0, a0, v, grad):
    """Broadcast on the host (numpy rules), evaluate on the device."""
    lib = _lib.load_library()
    arrs = np.broadcast_arrays(*[np.asarray(x, dtype=np.float64)
                                 for x in (R, t, p0, a0)])
    shape = arrs[0].shape
    dev = [torch.as_tensor(np.ascontiguousarray(x).reshape(-1),
                           device=_device()) for x in arrs]
    n = dev[0].numel()
    outs = [torch.empty(n, dtype=torch.float64, device=_device())
            for _ in range(3 if grad else 1)]
    if grad:
        args = (None, _lib.ptr(outs[0]), _lib.ptr(outs[1]), _lib.ptr(outs[2]))
    else:
        args = (_lib.ptr(outs[0]), None, None, None)
    _lib.check(lib.pc_pressure_kernel(*[_lib.ptr(x) for x in dev], n,
                                      float(v), *args, _lib.stream()),
               "pc_pressure_kernel")
    res = [o.cpu().numpy().reshape(shape) for o in outs]
    if len(shape) == 0:
        res = [float(x) for x in res]
    return res


def pressure_kernel(R, t, p0, a0, v):
    """Pressure radiated by one Gaussian ball, broadcasting over inputs
    (radiator.py:36-55; evaluated on the device in fp64)."""
    R = np.asarray(R, dtype=np.float64)
    if np.any(R <= 0):
        raise ValueError("source-sensor distance R must be > 0 "
                         "(sensor coincides with the ball center)")
    if not (np.all(np.asarray(a0) > 0) and v > 0):
        raise ValueError("a0 and v must be > 0")
    return _eval_pressure(R, t, p0, a0, v, grad=False)[0]


def pressure_kernel_grad(R, t, p0, a0, v):
    """Partials of pressure_kernel w.r.t. (p0, a0, R), broadcasting
    (radiator.py:58-83; evaluated on the device in fp64)."""
    R = np.asarray(R, dtype=np.float64)
    if np.any(R <= 0):
        raise ValueError("source-sensor distance R must be > 0")
    if not (np.all(np.asarray(a0) > 0) and v > 0):
        raise ValueError("a0 and v must be > 0")
    d_p0, d_a0, d_R = _eval_pressure(R, t, p0, a0, v, grad=True)
    return d_p0, d_a0, d_R


def _as_cloud_state(states):
    """radiator.py:177-183."""
    if isinstance(states, (list, tuple)):
        if all(isinstance(s, BallStateAtT) for s in states) or \
                all(hasattr(s, "a0_t") and np.ndim(s.a0_t) == 0
                    for s in states):
            return CloudState.from_states(states)
        raise TypeError("states must be a CloudState or a list of "
                        "BallStateAtT")
    if hasattr(states, "a0_t") and hasattr(states, "mu_t"):
        return states
    raise TypeError("states must be a CloudState or a list of BallStateAtT")


def _state_tensors(state):
    mu = to_device(state.mu_t, torch.float64).reshape(1, -1, 3)
    a0 = to_device(state.a0_t, torch.float32).reshape(1, -1)
    p0 = to_device(state.p0_t, torch.float32).reshape(1, -1)
    return mu, a0, p0


def _any_nonpositive(x) -> bool:
    if isinstance(x, torch.Tensor):
        return bool((x <= 0).any().item())
    return bool(np.any(np.asarray(x) <= 0))


def forward_frame(states, array, support_sigmas: float = DEFAULT_SUPPORT_SIGMAS,
                  exact: bool = False):
    """Superpose every ball's pressure trace at every sensor -> (M, T)."""
    state = _as_cloud_state(states)
    torch_io = _is_torch(state.a0_t, state.mu_t)
    darr = cached_device_array(array, support_sigmas, exact)
    B = len(state)
    if B == 0:
        z = torch.zeros((darr.M, darr.T), dtype=torch.float64,
                        device=_device())
        return z if torch_io else z.cpu().numpy()
    if _any_nonpositive(state.a0_t):
        raise ValueError("all a0_t must be > 0 (clamp before the radiator)")
    mu, a0, p0 = _state_tensors(state)
    out, _, coinc = forward_device(darr, mu, a0, p0)
    raise_if_coincident(coinc, mu, darr.positions)
    out = out[0].double()
    return out if torch_io else out.cpu().numpy()


def frame_state_grads(states, array, residual,
                      support_sigmas: float = DEFAULT_SUPPORT_SIGMAS,
                      exact: bool = False):
    """Gradient of 0.5*||residual||^2 w.r.t. (a0_t, p0_t, mu_t) -> (B, 5)."""
    state = _as_cloud_state(states)
    torch_io = _is_torch(state.a0_t, state.mu_t, residual)
    M, T = array.positions.shape[0], int(array.n_samples)
    if tuple(residual.shape) != (M, T):
        raise ValueError(
            f"residual shape {tuple(residual.shape)} does not match the "
            f"array ({M}, {T})")
    B = len(state)
    if B == 0:
        z = torch.zeros((0, 5), dtype=torch.float64, device=_device())
        return z if torch_io else z.cpu().numpy()
    darr = cached_device_array(array, support_sigmas, exact)
    mu, a0, p0 = _state_tensors(state)
    r = to_device(residual, torch.float32).reshape(1, M, T)
    G, coinc = state_grads_device(darr, mu, a0, p0, r)
    raise_if_coincident(coinc, mu, darr.positions)
    G = G[0].double()
    return G if torch_io else G.cpu().numpy()


def accumulate_frame_grads(states, state_grads, array, residual,
                           support_sigmas: float = DEFAULT_SUPPORT_SIGMAS,
                           exact: bool = False) -> CloudGrads:
    """Compose radiator and deformation partials into parameter gradients."""
    lib = _lib.load_library()
    state = _as_cloud_state(states)
    torch_io = _is_torch(state.a0_t, residual, state_grads.d_omega)
    M, T = array.positions.shape[0], int(array.n_samples)
    if tuple(residual.shape) != (M, T):
        raise ValueError(
            f"residual shape {tuple(residual.shape)} does not match the "
            f"array ({M}, {T})")
    sg = state_grads
    B, _, N = tuple(sg.d_omega.shape)
    dev = _device()
    shared = bool(sg.shared_basis)
    has_ts = sg.d_theta is not None and np.prod(sg.d_theta.shape) > 0
    if B == 0:
        G = torch.zeros((1, 0, 5), dtype=torch.float32, device=dev)
    else:
        darr = cached_device_array(array, support_sigmas, exact)
        mu, a0, p0 = _state_tensors(state)
        r = to_device(residual, torch.float32).reshape(1, M, T)
        G, coinc = state_grads_device(darr, mu, a0, p0, r)
        raise_if_coincident(coinc, mu, darr.positions)
    d_base = to_device(sg.d_base, torch.float64)
    d_om = to_device(sg.d_omega, torch.float64)
    d_th = to_device(sg.d_theta, torch.float64) if has_ts else None
    d_sg = to_device(sg.d_sigma, torch.float64) if has_ts else None
    f64 = dict(dtype=torch.float64, device=dev)
    g_p0 = torch.zeros(B, **f64)
    g_a0 = torch.zeros(B, **f64)
    g_mu = torch.zeros((B, 3), **f64)
    ts_shape = ((B, N) if shared else (B, 5, N)) if has_ts else (B, 0)
    g_th = torch.zeros(ts_shape, **f64)
    g_sg = torch.zeros(ts_shape, **f64)
    g_om = torch.zeros((B, 5, N), **f64)
    rows = _lib.i32_array(np.asarray(sg.omega_row).ravel()[:5])
    _lib.check(lib.pc_assemble_grads(
        _lib.ptr(G), B, N, _lib.ptr(d_base), _lib.ptr(d_om), _lib.ptr(d_th),
        _lib.ptr(d_sg), rows, int(shared), int(has_ts), _lib.ptr(g_p0),
        _lib.ptr(g_a0), _lib.ptr(g_mu), _lib.ptr(g_th), _lib.ptr(g_sg),
        _lib.ptr(g_om), _lib.stream()), "pc_assemble_grads")
    out = [g_p0, g_a0, g_mu, g_th, g_sg, g_om]
    if not torch_io:
        out = [x.cpu().numpy() for x in out]
    return CloudGrads(*out)
