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
    """Unit-sum separable Gaussian window (size x size)."""
    half = (size - 1) / 2.0
    g1 = np.exp(-0.5 * ((np.arange(size) - half) / sigma) ** 2)
    g1 /= g1.sum()
    return np.outer(g1, g1)


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
    x, y = torch.as_tensor(av, device=dev), torch.as_tensor(bv, device=dev)
    win = torch.as_tensor(gaussian_window(), device=dev)
    stab1, stab2 = (SSIM_K1 * data_range) ** 2, (SSIM_K2 * data_range) ** 2
    # local moments: E[x], E[y], E[x^2], E[y^2], E[xy] over each window
    ex, ey, exx, eyy, exy = (_window_mean(t, win)
                             for t in (x, y, x * x, y * y, x * y))
    luminance = (2.0 * ex * ey + stab1) / (ex * ex + ey * ey + stab1)
    structure = (2.0 * (exy - ex * ey) + stab2) / \
        ((exx - ex * ex) + (eyy - ey * ey) + stab2)
    return float((luminance * structure).mean().item())


def eval_report(recon_grids, truth_grids, ubp_grids=None) -> list:
    """Per-frame, per-axis SSIM of MAP images against ground truth, methods
    "4d" (and "ubp"), each pair normalised by its joint maximum."""
    truth = list(truth_grids)
    runs = [("4d", list(recon_grids))]
    if ubp_grids is not None:
        runs.append(("ubp", list(ubp_grids)))
    for name, grids in runs:
        if len(grids) != len(truth):
            what = "recon" if name == "4d" else name
            raise ValueError(f"frame counts of {what} and truth differ")
    return [{"frame": k, "axis": ax, "method": name,
             "ssim": ssim(*normalize_pair(map_project(grids[k], ax),
                                          map_project(truth[k], ax)))}
            for k in range(len(truth)) for ax in MAP_AXES
            for name, grids in runs]


def format_report(records) -> str:
    """Aligned text table of an eval_report result."""
    table = {(r["frame"], r["axis"], r["method"]): r["ssim"] for r in records}
    methods = sorted({m for _, _, m in table})
    header = [f"{m}/{ax}" for m in methods for ax in MAP_AXES]
    out = ["frame  " + "  ".join(h.rjust(10) for h in header)]
    for k in sorted({f for f, _, _ in table}):
        row = [table[(k, ax, m)] for m in methods for ax in MAP_AXES]
        out.append(f"{k:5d}  " + "  ".join(f"{v:10.4f}" for v in row))
    return "\n".join(out)
