"""Voxelisation, maximum-amplitude projections and SSIM.

Mirrors pacloud/evaluation.py: ``GridSpec`` (:22-43), ``voxelize``
(:77-93, the numba ``_splat_balls`` :46-74 becomes ``pc_voxelize``),
``MapImage`` / ``map_project`` (:96-119), ``normalize_pair`` (:126-139),
``gaussian_window`` (:142-148), ``ssim`` (:157-184), ``eval_report``
(:187-216) and ``format_report`` (:219-230).

Grids are computed on the GPU (deterministic, fp32 accumulation); MAP and
SSIM run on the device in fp64 with torch (valid 11x11 Gaussian-window
statistics, the reference's constants), so a reconstruction is scored
without leaving the GPU until the final scalars.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import Box, CloudState, VoxelGrid
from .radiator import DEFAULT_SUPPORT_SIGMAS, _device

MAP_AXES = ("XY", "YZ", "XZ")
_DROP = {"XY": 2, "YZ": 0, "XZ": 1}     # axis removed by each projection

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03


@dataclass(frozen=True)
class GridSpec:
    """Voxel grid geometry; `origin` is the centre of voxel (0, 0, 0)."""

    origin: np.ndarray
    spacing: float
    dims: tuple

    def __post_init__(self):
        o = np.asarray(self.origin, dtype=np.float64)
        if o.shape != (3,):
            raise ValueError("origin must be a 3-vector")
        object.__setattr__(self, "origin", o)
        object.__setattr__(self, "dims", tuple(int(d) for d in self.dims))
        if not self.spacing > 0:
            raise ValueError("spacing must be > 0")

    @classmethod
    def from_box(cls, box: Box, spacing: float) -> "GridSpec":
        dims = tuple(max(1, int(np.round(s / spacing))) for s in box.size)
        return cls(box.lo + 0.5 * spacing, spacing, dims)


def _state_arrays(states):
    if isinstance(states, (list, tuple)):
        states = CloudState.from_states(states)
    return (np.ascontiguousarray(states.mu_t, dtype=np.float64).reshape(-1, 3),
            np.ascontiguousarray(states.a0_t, dtype=np.float64).ravel(),
            np.ascontiguousarray(states.p0_t, dtype=np.float64).ravel())


def voxelize_device(mu, a0, p0, spec: GridSpec,
                    support_sigmas: float = DEFAULT_SUPPORT_SIGMAS,
                    exact: bool = False) -> torch.Tensor:
    """pc_voxelize: (nx, ny, nz) float32 on the device from device (B,3) /
    (B,) / (B,) float64 tensors."""
    lib = _lib.load_library()
    dev = mu.device if isinstance(mu, torch.Tensor) else _device()
    mu = torch.as_tensor(mu, dtype=torch.float64, device=dev).reshape(-1, 3).contiguous()
    a0 = torch.as_tensor(a0, dtype=torch.float64, device=dev).reshape(-1).contiguous()
    p0 = torch.as_tensor(p0, dtype=torch.float64, device=dev).reshape(-1).contiguous()
    B = a0.numel()
    out = torch.empty(spec.dims, dtype=torch.float32, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib.pc_voxelize_workspace_bytes(B)), dtype=torch.uint8,
                     device=dev)
    origin = (ctypes.c_double * 3)(*spec.origin.tolist())
    dims = (ctypes.c_int32 * 3)(*spec.dims)
    _lib.check(lib.pc_voxelize(
        _lib.ptr(mu), _lib.ptr(a0), _lib.ptr(p0), B, origin,
        float(spec.spacing), dims, float(support_sigmas), int(bool(exact)),
        _lib.ptr(out), _lib.ptr(bad), _lib.ptr(ws), ws.numel(), _lib.stream()),
        "pc_voxelize")
    if B and int(bad.item()):
        raise ValueError("all a0_t must be > 0")
    return out


def voxelize(states, spec: GridSpec,
             support_sigmas: float = DEFAULT_SUPPORT_SIGMAS,
             exact: bool = False) -> VoxelGrid:
    """Sample the cloud's Gaussian field at the voxel centres (reference
    signature; float64 VoxelGrid on the host)."""
    mu, a0, p0 = _state_arrays(states)
    if len(a0) and (a0 <= 0).any():
        raise ValueError("all a0_t must be > 0")
    vals = voxelize_device(mu, a0, p0, spec, support_sigmas, exact)
    return VoxelGrid(spec.origin, spec.spacing, spec.dims,
                     vals.double().cpu().numpy())


@dataclass(frozen=True)
class MapImage:
    """Maximum-amplitude projection of a grid along one axis."""

    values: np.ndarray
    axis: str
    pitch: float

    def __post_init__(self):
        if self.axis not in MAP_AXES:
            raise ValueError(f"axis must be one of {MAP_AXES}")
        v = np.asarray(self.values, dtype=np.float64)
        if v.ndim != 2:
            raise ValueError("map image values must be 2-d")
        object.__setattr__(self, "values", v)


def _values(x):
    if isinstance(x, MapImage):
        return x.values
    if isinstance(x, VoxelGrid):
        return x.values
    return x if isinstance(x, torch.Tensor) else np.asarray(x, np.float64)


def map_project(grid, axis: str) -> MapImage:
    """Per-pixel maximum along the dropped axis (VoxelGrid or tensor)."""
    if axis not in MAP_AXES:
        raise ValueError(f"axis must be one of {MAP_AXES}")
    v = _values(grid)
    pitch = grid.spacing if isinstance(grid, VoxelGrid) else 1.0
    if isinstance(v, torch.Tensor):
        return MapImage(torch.amax(v, dim=_DROP[axis]).double().cpu().numpy(),
                        axis, pitch)
    return MapImage(np.max(v, axis=_DROP[axis]), axis, pitch)


def normalize_pair(a, b):
    """Scale both images by their joint maximum (unchanged if it is <= 0)."""
    av = np.asarray(_values(a), np.float64)
    bv = np.asarray(_values(b), np.float64)
    peak = max(float(av.max()), float(bv.max()))
    if peak <= 0:
        return av, bv
    return av / peak, bv / peak


def gaussian_window(size: int = SSIM_WINDOW,
                    sigma: float = SSIM_SIGMA) -> np.ndarray:
    r = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    g = np.exp(-0.5 * (r / sigma) ** 2)
    w = np.outer(g, g)
    return w / w.sum()


def _window_mean(img: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """Valid 2-d correlation with the window (full windows only)."""
    return torch.nn.functional.conv2d(img[None, None], w[None, None])[0, 0]


def ssim(a, b, data_range: float = 1.0) -> float:
    """Mean local SSIM over fully contained 11x11 Gaussian windows
    (sigma 1.5, K1 0.01, K2 0.03); inputs on a [0, 1] scale."""
    av = np.asarray(_values(a), np.float64)
    bv = np.asarray(_values(b), np.float64)
    if av.shape != bv.shape:
        raise ValueError(f"image shapes differ: {av.shape} vs {bv.shape}")
    if min(av.shape) < SSIM_WINDOW:
        raise ValueError(
            f"images must be at least {SSIM_WINDOW} pixels per side")
    dev = _device() if torch.cuda.is_available() else torch.device("cpu")
    ta = torch.as_tensor(av, device=dev)
    tb = torch.as_tensor(bv, device=dev)
    w = torch.as_tensor(gaussian_window(), device=dev)
    c1 = (SSIM_K1 * data_range) ** 2
    c2 = (SSIM_K2 * data_range) ** 2
    mu_a, mu_b = _window_mean(ta, w), _window_mean(tb, w)
    var_a = _window_mean(ta * ta, w) - mu_a * mu_a
    var_b = _window_mean(tb * tb, w) - mu_b * mu_b
    cov = _window_mean(ta * tb, w) - mu_a * mu_b
    num = (2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2)
    den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2)
    return float((num / den).mean().item())


def eval_report(recon_grids, truth_grids, ubp_grids=None) -> list:
    """Per-frame, per-axis SSIM of MAP images against ground truth, methods
    "4d" (and "ubp"), each pair normalised by its joint maximum."""
    recon_grids, truth_grids = list(recon_grids), list(truth_grids)
    if len(recon_grids) != len(truth_grids):
        raise ValueError("frame counts of recon and truth differ")
    methods = {"4d": recon_grids}
    if ubp_grids is not None:
        ubp_grids = list(ubp_grids)
        if len(ubp_grids) != len(truth_grids):
            raise ValueError("frame counts of ubp and truth differ")
        methods["ubp"] = ubp_grids
    out = []
    for k, truth in enumerate(truth_grids):
        for axis in MAP_AXES:
            t_map = map_project(truth, axis)
            for name, grids in methods.items():
                rn, tn = normalize_pair(map_project(grids[k], axis), t_map)
                out.append({"frame": k, "axis": axis, "method": name,
                            "ssim": ssim(rn, tn)})
    return out


def format_report(records) -> str:
    """Aligned text table of an eval_report result."""
    methods = sorted({r["method"] for r in records})
    frames = sorted({r["frame"] for r in records})
    val = {(r["frame"], r["axis"], r["method"]): r["ssim"] for r in records}
    cols = [f"{m}/{ax}" for m in methods for ax in MAP_AXES]
    lines = ["frame  " + "  ".join(f"{c:>10s}" for c in cols)]
    for k in frames:
        lines.append(f"{k:5d}  " + "  ".join(
            f"{val[(k, ax, m)]:10.4f}" for m in methods for ax in MAP_AXES))
    return "\n".join(lines)
