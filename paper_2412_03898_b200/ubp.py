"""Universal back-projection comparator on the GPU.

Mirrors pacloud/reconstruction.py:380-417 ``ubp_reconstruct``: the same
window-coverage check and error message on the host, then pc_ubp_filter
(b = 2 p - 2 t dp/dt) and pc_backproject (voxel-major gather, linear
interpolation at each voxel's time of flight) on the device.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import VoxelGrid
from .radiator import _device


def _check_window(array, spec):
    """reconstruction.py:391-396: the sample window must cover every
    voxel's time of flight."""
    times = array.sample_times()
    lo = spec.origin
    hi = spec.origin + spec.spacing * (np.array(spec.dims) - 1)
    bits = (np.arange(8)[:, None] >> np.arange(3)[None, :]) & 1
    corners = np.where(bits == 0, lo, hi)
    pos = array.positions
    d_corner = np.linalg.norm(pos[:, None, :] - corners[None, :, :], axis=2)
    d_near = np.linalg.norm(pos - np.clip(pos, lo, hi), axis=1)
    tof_min = float(np.min(d_near)) / array.sound_speed
    tof_max = float(np.max(d_corner)) / array.sound_speed
    if tof_min < times[0] or tof_max > times[-1]:
        raise ValueError(
            f"sample window [{times[0]:.3f}, {times[-1]:.3f}] us does not "
            f"cover voxel times of flight [{tof_min:.3f}, {tof_max:.3f}] us "
            f"(shortfall {max(0.0, times[0] - tof_min):.3f} us before, "
            f"{max(0.0, tof_max - times[-1]):.3f} us after)")


def ubp_device(traces, array, spec) -> torch.Tensor:
    """(nx, ny, nz) float32 back-projection on the device; traces (M, T)
    numpy or device tensor."""
    lib = _lib.load_library()
    dev = traces.device if isinstance(traces, torch.Tensor) else _device()
    tr = torch.as_tensor(traces, dtype=torch.float64, device=dev).contiguous()
    M, T = array.n_sensors, array.n_samples
    if tuple(tr.shape) != (M, T):
        raise ValueError(f"traces shape {tuple(tr.shape)} does not match the "
                         f"array")
    _check_window(array, spec)
    filt = torch.empty((M, T), dtype=torch.float32, device=dev)
    _lib.check(lib.pc_ubp_filter(_lib.ptr(tr), M, T, float(array.t_start),
                                 float(array.sample_rate), _lib.ptr(filt),
                                 _lib.stream()), "pc_ubp_filter")
    pos = torch.as_tensor(array.positions, dtype=torch.float64,
                          device=dev).contiguous()
    out = torch.empty(spec.dims, dtype=torch.float32, device=dev)
    origin = (ctypes.c_double * 3)(*np.asarray(spec.origin, float).tolist())
    dims = (ctypes.c_int32 * 3)(*spec.dims)
    _lib.check(lib.pc_backproject(
        _lib.ptr(filt), _lib.ptr(pos), M, T, float(array.sound_speed),
        float(array.t_start), float(array.dt), origin, float(spec.spacing),
        dims, _lib.ptr(out), _lib.stream()), "pc_backproject")
    return out


def ubp_reconstruct(traces, array, spec) -> VoxelGrid:
    """Universal back-projection of one frame (reference signature)."""
    if not isinstance(traces, torch.Tensor):
        traces = np.ascontiguousarray(traces, dtype=np.float64)
    vals = ubp_device(traces, array, spec)
    return VoxelGrid(spec.origin, spec.spacing, spec.dims,
                     vals.double().cpu().numpy())
