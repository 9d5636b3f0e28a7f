"""Drop-in optimisation engine calls on the B200.

Mirrors pkg/src/pacloud/reconstruction.py: ``l2_loss`` (:28-35),
``scheduled_lr`` (:38-41), ``AdamState`` / ``adam_step`` (:44-69),
``sgd_step`` (:72-76), ``ParamGroup`` / ``ParamGroups`` (:79-134) and
``dynamic_reconstruct`` (:253-336), same signatures and exceptions.  The
arithmetic runs in libpacloud_b200.so (pc_l2_loss, pc_check_finite,
pc_adam_segments, pc_sgd_segments, pc_gather_rows); ``dynamic_reconstruct``
drives the fused ``IterationEngine``.
"""

from __future__ import annotations

import math
import warnings

import numpy as np
import torch

from . import _lib
from .core import AdamState, DynamicCloud
from .engine import (GROUP_ORDER, IterationEngine, identity_cloud,
                     scheduled_lr, select_frames)
from .radiator import _device, _is_torch, to_device

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8

__all__ = ["l2_loss", "scheduled_lr", "AdamState", "adam_step", "sgd_step",
           "ParamGroup", "ParamGroups", "dynamic_reconstruct",
           "ADAM_BETA1", "ADAM_BETA2", "ADAM_EPS"]


def l2_loss(predicted, observed) -> float:
    """0.5 * sum of squared differences over all entries."""
    lib = _lib.load_library()
    if tuple(np.shape(predicted)) != tuple(np.shape(observed)):
        raise ValueError(f"shape mismatch: {tuple(np.shape(predicted))} vs "
                         f"{tuple(np.shape(observed))}")
    p = to_device(predicted, torch.float64).reshape(-1)
    o = to_device(observed, torch.float64).reshape(-1)
    out = torch.zeros(1, dtype=torch.float64, device=p.device)
    _lib.check(lib.pc_l2_loss(_lib.ptr(p), _lib.ptr(o), p.numel(),
                              _lib.ptr(out), _lib.stream()), "pc_l2_loss")
    return float(out.item())


def _finite_or_raise(g: torch.Tensor, group: str) -> None:
    """reconstruction.py:60-61 on the caller's float64 gradient."""
    lib = _lib.load_library()
    flags = torch.zeros(1, dtype=torch.int32, device=g.device)
    _lib.check(lib.pc_check_finite_f64(
        _lib.ptr(g), 1, _lib.i64_array([0, g.numel()]), _lib.ptr(flags),
        _lib.stream()), "pc_check_finite_f64")
    if int(flags.item()):
        raise ValueError(f"non-finite gradient in parameter group '{group}'")


def _inplace(param, dev_value: torch.Tensor) -> None:
    if isinstance(param, torch.Tensor):
        param.copy_(dev_value.reshape(param.shape))
    else:
        param[...] = dev_value.reshape(param.shape).cpu().numpy()


def adam_step(param, grad, state: AdamState, lr: float,
              group: str = "") -> None:
    """One in-place Adam update (beta1 0.9, beta2 0.999, eps 1e-8), in
    float64 like reconstruction.py:57-69 (pc_adam_segments_f64)."""
    lib = _lib.load_library()
    g = to_device(grad, torch.float64).reshape(-1)
    if g.numel() != int(np.prod(np.shape(param))):
        raise ValueError("grad and param sizes differ")
    _finite_or_raise(g, group)
    p = to_device(param, torch.float64).reshape(-1).clone()
    m = to_device(state.m, torch.float64).reshape(-1).clone()
    v = to_device(state.v, torch.float64).reshape(-1).clone()
    state.t += 1
    if p.numel():
        _lib.check(lib.pc_adam_segments_f64(
            _lib.ptr(p), _lib.ptr(g), _lib.ptr(m), _lib.ptr(v), 1,
            _lib.i64_array([0, p.numel()]), _lib.f64_array([lr]),
            _lib.i32_array([state.t]), _lib.f64_array([-math.inf]),
            _lib.stream()), "pc_adam_segments_f64")
    _inplace(param, p)
    _inplace(state.m, m)
    _inplace(state.v, v)


def sgd_step(param, grad, lr: float, group: str = "") -> None:
    """reconstruction.py:72-76 in float64 (pc_sgd_segments_f64)."""
    lib = _lib.load_library()
    g = to_device(grad, torch.float64).reshape(-1)
    _finite_or_raise(g, group)
    p = to_device(param, torch.float64).reshape(-1).clone()
    if p.numel():
        _lib.check(lib.pc_sgd_segments_f64(
            _lib.ptr(p), _lib.ptr(g), 1, _lib.i64_array([0, p.numel()]),
            _lib.f64_array([lr]), _lib.f64_array([-math.inf]),
            _lib.stream()), "pc_sgd_segments_f64")
    _inplace(param, p)


def gather_rows(arr, index: torch.Tensor):
    """Stable row gather on the device (pc_gather_rows)."""
    lib = _lib.load_library()
    torch_io = _is_torch(arr)
    src = to_device(arr, torch.float64)
    n = int(index.numel())
    dst = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype,
                      device=src.device)
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 0
    if n and row_bytes:
        _lib.check(lib.pc_gather_rows(_lib.ptr(src), _lib.ptr(dst),
                                      _lib.ptr(index), n, row_bytes,
                                      _lib.stream()), "pc_gather_rows")
    return dst if torch_io else dst.cpu().numpy()


def keep_index(keep) -> torch.Tensor:
    """Stable survivor index of a boolean mask (pc_compact_index)."""
    lib = _lib.load_library()
    k = to_device(np.asarray(keep, dtype=np.uint8) if not _is_torch(keep)
                  else keep.to(torch.uint8), torch.uint8).reshape(-1)
    B = int(k.numel())
    dev = k.device
    ws = torch.empty(int(lib.pc_compact_workspace_bytes(B)), dtype=torch.uint8,
                     device=dev)
    idx = torch.empty(max(B, 1), dtype=torch.int64, device=dev)
    n_out = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(lib.pc_compact_index(_lib.ptr(k), None, B, _lib.ptr(idx),
                                    _lib.ptr(n_out), _lib.ptr(ws), ws.numel(),
                                    _lib.stream()), "pc_compact_index")
    return idx[:int(n_out.item())]


class ParamGroup:
    """Named set of parameter arrays sharing one learning rate."""

    def __init__(self, name: str, lr0: float, params: dict):
        self.name = name
        self.lr0 = lr0
        self.params = params
        self.adam = {k: AdamState.like(p) for k, p in params.items()}

    def step(self, grads: dict, lr: float, optimizer: str):
        for key, param in self.params.items():
            if optimizer == "adam":
                adam_step(param, grads[key], self.adam[key], lr, self.name)
            else:
                sgd_step(param, grads[key], lr, self.name)

    def prune(self, keep):
        """Drop balls along the leading axis of every array and its moments
        (reconstruction.py:95-100), gathering on the device."""
        idx = keep_index(keep)
        for key in self.params:
            self.params[key] = gather_rows(self.params[key], idx)
            st = self.adam[key]
            self.adam[key] = AdamState(gather_rows(st.m, idx),
                                       gather_rows(st.v, idx), st.t)


class ParamGroups:
    """The four optimiser groups: coords, pressure, std, deform."""

    ORDER = ("coords", "pressure", "std", "deform")

    def __init__(self, groups: dict):
        if set(groups) != set(self.ORDER):
            raise ValueError(f"groups must be exactly {self.ORDER}")
        seen: set[int] = set()
        for g in groups.values():
            for p in g.params.values():
                if id(p) in seen:
                    raise ValueError(
                        "a parameter array appears in more than one group")
                seen.add(id(p))
        self.groups = groups

    def __getitem__(self, name: str) -> ParamGroup:
        return self.groups[name]

    def lrs_at(self, iteration: int, step_size: int,
               drop_rate: float) -> dict:
        return {name: scheduled_lr(g.lr0, iteration, step_size, drop_rate)
                for name, g in self.groups.items()}

    def prune(self, keep):
        for g in self.groups.values():
            g.prune(keep)


def observed_frame_major(observed) -> torch.Tensor:
    """SignalSet data (M, K, T) -> device float32 (K, M, T)."""
    data = observed.data if hasattr(observed, "data") else observed
    t = to_device(data, torch.float32)
    return t.permute(1, 0, 2).contiguous()


def dynamic_reconstruct(observed, array, init_balls, config, roi=None,
                        progress=None) -> DynamicCloud:
    """Fit deformation fields and baseline attributes to all frames.

    Same contract as reconstruction.py:253-336; every iteration runs on the
    device through IterationEngine (one host sync per iteration).
    """
    init_balls = list(init_balls)
    if not init_balls:
        raise ValueError("init cloud must be nonempty")
    if observed.n_frames < 2:
        raise ValueError("dynamic reconstruction needs at least 2 frames")
    observed.validate_against(array)
    basis = getattr(config, "basis", "gauss")
    nb = config.n_basis if basis == "gauss" else \
        getattr(config, "n_basis_pf", 8)
    p0 = np.array([b.p0 for b in init_balls], dtype=np.float64)
    a0 = np.array([b.a0 for b in init_balls], dtype=np.float64)
    mu = np.array([b.mu for b in init_balls], dtype=np.float64)
    cloud = identity_cloud(p0, a0, mu, nb, basis)
    eng = IterationEngine(cloud, array, observed_frame_major(observed),
                          observed.frame_times, config)
    eng.stage_timing = progress is not None
    rng = np.random.default_rng(config.seed)
    for it in range(config.dynamic_iters):
        frames = select_frames(observed.n_frames, config.frame_batch, rng)
        loss = eng.iterate(it, frames)
        if progress is not None:
            # the reference's record (reconstruction.py:329-332) plus the
            # device stage timings of this iteration (CUDA events)
            progress({"stage": "dynamic", "iteration": it, "loss": loss,
                      "n_balls": eng.B,
                      "frames": [int(k) for k in frames],
                      **{f"lr_{k}": v for k, v in eng.last_lrs.items()},
                      **(eng.last_timing or {})})
    out = eng.cloud()
    if roi is not None:
        _warn_outside_roi(out, roi, observed.frame_times, config)
    return out


def _warn_outside_roi(cloud, roi, times, config):
    """reconstruction.py:339-349 (states from the device kernel)."""
    from .deformation import cloud_states_at
    worst = 0
    for t in times:
        st = cloud_states_at(cloud, float(t), config.coord_mode,
                             a0_floor=config.a0_floor)
        worst = max(worst, int(np.sum(~roi.contains(st.mu_t))))
    if worst:
        warnings.warn(
            f"{worst} ball(s) drift outside the region of interest at some "
            f"frame time", RuntimeWarning, stacklevel=3)
