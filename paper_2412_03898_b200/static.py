"""Static stage on the B200.

Mirrors pacloud/reconstruction.py:160-231 ``static_reconstruct``: a uniform
lattice over the ROI (pitch init_pitch, a0 = pitch / 2, p0 = init_p0_scale x
data peak) fitted to one frame by Adam (or SGD) on (p0, a0, mu), groups in
the reference's order pressure -> std -> coords, floors after the step, and
every prune_every iterations the balls with p0 <= prune_threshold x max(p0)
dropped together with their Adam moments (step counts kept).

``StaticEngine`` keeps the parameters, gradients and moments in one flat
device buffer [p0 | a0 | mu] and runs forward + fused loss
(pc_forward_traces), adjoint (pc_residual_state_grads), the finite guard
(pc_check_finite) and the three group updates in one pc_adam_segments
launch, with one host sync per iteration; pruning compacts on the device
(pc_prune_mask / pc_compact_index / pc_gather_rows).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .core import GaussBall
from .engine import scheduled_lr
from .geometry import box_lattice
from .radiator import (DeviceArray, _device, forward_device,
                       raise_if_coincident, state_grads_device)

# (segment, group, reference ParamGroup order of the step calls)
STATIC_SEGMENTS = (("p0", "pressure"), ("a0", "std"), ("mu", "coords"))


class StaticEngine:
    """Single-frame fit of a static cloud, device resident."""

    def __init__(self, p0, a0, mu, array, observed, config, device=None):
        self.cfg = config
        self.device = device or _device()
        dev = self.device
        p0 = np.asarray(p0, np.float64).reshape(-1)
        a0 = np.asarray(a0, np.float64).reshape(-1)
        mu = np.asarray(mu, np.float64).reshape(-1, 3)
        obs = observed.detach() if isinstance(observed, torch.Tensor) else \
            torch.as_tensor(np.ascontiguousarray(observed, np.float32))
        if tuple(obs.shape) != (array.n_sensors, array.n_samples):
            raise ValueError(
                f"observed shape {tuple(obs.shape)} does not match the array")
        self.obs = obs.to(dev, torch.float32).reshape(1, array.n_sensors,
                                                     array.n_samples).contiguous()
        self.darr = DeviceArray(array, config.support_sigmas,
                                config.exact_forward)
        self.steps = {name: 0 for name, _ in STATIC_SEGMENTS}
        self._alloc(len(p0))
        self.P[:self.B] = torch.as_tensor(p0, device=dev)
        self.P[self.B:2 * self.B] = torch.as_tensor(a0, device=dev)
        self.P[2 * self.B:] = torch.as_tensor(mu.ravel(), device=dev)
        self.Mo.zero_()
        self.Vo.zero_()

    # ------------------------------------------------------------ buffers
    def _alloc(self, B: int):
        dev, M, T = self.device, self.darr.M, self.darr.T
        self.B = B
        f64 = dict(dtype=torch.float64, device=dev)
        self.P = torch.empty(5 * B, **f64)
        self.Mo = torch.empty(5 * B, **f64)
        self.Vo = torch.empty(5 * B, **f64)
        self.Gf = torch.zeros(5 * B, dtype=torch.float32, device=dev)
        self.a0_t = torch.empty((1, B), dtype=torch.float32, device=dev)
        self.p0_t = torch.empty((1, B), dtype=torch.float32, device=dev)
        self.resid = torch.empty((1, M, T), dtype=torch.float32, device=dev)
        self.G = torch.empty((1, B, 5), dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.flags = torch.zeros(3, dtype=torch.int32, device=dev)
        self.coinc = torch.full((1,), _lib.INT64_MAX, dtype=torch.int64,
                                device=dev)
        self.ws = torch.empty(max(self.darr.workspace_bytes(max(B, 1), 1), 1),
                              dtype=torch.uint8, device=dev)
        self.offsets = [0, B, 2 * B, 5 * B]

    @property
    def p0(self):
        return self.P[:self.B]

    @property
    def a0(self):
        return self.P[self.B:2 * self.B]

    @property
    def mu(self):
        return self.P[2 * self.B:].view(self.B, 3)

    # ------------------------------------------------------------ iteration
    def _grads(self):
        B = self.B
        self.coinc.fill_(_lib.INT64_MAX)
        self.a0_t[0].copy_(self.a0)
        self.p0_t[0].copy_(self.p0)
        mu_t = self.mu.view(1, B, 3)
        forward_device(self.darr, mu_t, self.a0_t, self.p0_t,
                       observed=self.obs, out=self.resid, loss=self.loss,
                       coincident=self.coinc, workspace=self.ws)
        state_grads_device(self.darr, mu_t, self.a0_t, self.p0_t, self.resid,
                           G=self.G, coincident=self.coinc)
        g = self.G[0]
        self.Gf[:B].copy_(g[:, 1])
        self.Gf[B:2 * B].copy_(g[:, 0])
        self.Gf[2 * B:].view(B, 3).copy_(g[:, 2:5])

    def _update(self, names, lrs):
        lib = _lib.load_library()
        cfg = self.cfg
        floors = {"p0": cfg.p0_floor, "a0": cfg.a0_floor, "mu": -math.inf}
        idx = [i for i, (n, _) in enumerate(STATIC_SEGMENTS) if n in names]
        if not idx:
            return
        for i in idx:
            self.steps[STATIC_SEGMENTS[i][0]] += 1
        for i in idx:          # one launch per segment keeps the offsets simple
            name, group = STATIC_SEGMENTS[i]
            off = _lib.i64_array([self.offsets[i], self.offsets[i + 1]])
            if cfg.optimizer == "adam":
                _lib.check(lib.pc_adam_segments(
                    _lib.ptr(self.P), _lib.ptr(self.Gf), _lib.ptr(self.Mo),
                    _lib.ptr(self.Vo), 1, off, _lib.f64_array([lrs[group]]),
                    _lib.i32_array([self.steps[name]]),
                    _lib.f64_array([floors[name]]), _lib.stream()),
                    "pc_adam_segments")
            else:
                _lib.check(lib.pc_sgd_segments(
                    _lib.ptr(self.P), _lib.ptr(self.Gf), 1, off,
                    _lib.f64_array([lrs[group]]),
                    _lib.f64_array([floors[name]]), _lib.stream()),
                    "pc_sgd_segments")

    def iterate(self, it: int):
        """One iteration; returns (loss, lrs) like the reference loop body
        (reconstruction.py:190-218, before the prune check)."""
        lib = _lib.load_library()
        cfg = self.cfg
        lrs = {g: scheduled_lr(getattr(cfg, "lr_" + k), it, cfg.step_size,
                               cfg.drop_rate)
               for g, k in (("coords", "coords"), ("pressure", "pressure"),
                            ("std", "std"), ("deform", "deform"))}
        self._grads()
        self.flags.zero_()
        _lib.check(lib.pc_check_finite(
            _lib.ptr(self.Gf), 3, _lib.i64_array(self.offsets),
            _lib.ptr(self.flags), _lib.stream()), "pc_check_finite")
        status = torch.cat([self.loss, self.flags.double(),
                            self.coinc.double()]).cpu().numpy()
        loss = float(status[0])
        if status[4] < 9.0e18:
            raise_if_coincident(int(status[4]), self.mu, self.darr.positions)
        if not math.isfinite(loss):
            raise RuntimeError(f"non-finite loss at iteration {it}")
        done = []
        for i, (name, group) in enumerate(STATIC_SEGMENTS):
            if status[1 + i]:
                self._update(done, lrs)
                raise ValueError(
                    f"non-finite gradient in parameter group '{group}'")
            done.append(name)
        self._update(done, lrs)
        return loss, lrs

    def prune(self) -> int:
        """keep = p0 > prune_threshold * max(p0, initial=0)
        (reconstruction.py:219-226); returns the survivor count."""
        lib = _lib.load_library()
        B, dev = self.B, self.device
        keep = torch.empty(B, dtype=torch.uint8, device=dev)
        count = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(int(lib.pc_compact_workspace_bytes(B)),
                         dtype=torch.uint8, device=dev)
        _lib.check(lib.pc_prune_mask(
            _lib.ptr(self.p0), B, float(self.cfg.prune_threshold),
            _lib.ptr(keep), _lib.ptr(count), _lib.ptr(ws), ws.numel(),
            _lib.stream()), "pc_prune_mask")
        n = int(count.item())
        if n == 0:
            raise RuntimeError("all balls pruned; lower recon.prune_threshold "
                               "or check the input data")
        if n == B:
            return B
        index = torch.empty(B, dtype=torch.int64, device=dev)
        n_out = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(lib.pc_compact_index(
            _lib.ptr(keep), None, B, _lib.ptr(index), _lib.ptr(n_out),
            _lib.ptr(ws), ws.numel(), _lib.stream()), "pc_compact_index")
        index = index[:n]
        old = (self.P, self.Mo, self.Vo)
        old_off = list(self.offsets)
        self._alloc(n)
        for src, dst in zip(old, (self.P, self.Mo, self.Vo)):
            for i in range(3):
                row = (old_off[i + 1] - old_off[i]) // B * 8
                _lib.check(lib.pc_gather_rows(
                    _lib.ptr(src[old_off[i]:]),
                    _lib.ptr(dst[self.offsets[i]:]), _lib.ptr(index), n, row,
                    _lib.stream()), "pc_gather_rows")
        return n

    def balls(self) -> list:
        p0 = self.p0.cpu().numpy()
        a0 = self.a0.cpu().numpy()
        mu = self.mu.cpu().numpy()
        return [GaussBall(p0[i], a0[i], mu[i]) for i in range(len(p0))]


def initial_lattice(observed, roi, config):
    """reconstruction.py:170-177: lattice centres, a0 = pitch / 2, p0 =
    init_p0_scale x max |observed|."""
    mu = box_lattice(roi, config.init_pitch)
    obs = observed.detach().abs().max().item() if isinstance(
        observed, torch.Tensor) else (float(np.max(np.abs(observed)))
                                      if np.size(observed) else 0.0)
    return (np.full(len(mu), config.init_p0_scale * float(obs)),
            np.full(len(mu), config.init_pitch / 2.0), mu)


def static_reconstruct(observed, array, config, roi, progress=None) -> list:
    """Fit a static ball cloud to one reference frame (same contract and
    exceptions as reconstruction.py:160-231); returns a list of GaussBall."""
    if not isinstance(observed, torch.Tensor):
        observed = np.ascontiguousarray(observed, dtype=np.float64)
    if tuple(observed.shape) != (array.n_sensors, array.n_samples):
        raise ValueError(
            f"observed shape {tuple(observed.shape)} does not match the array")
    p0, a0, mu = initial_lattice(observed, roi, config)
    eng = StaticEngine(p0, a0, mu, array, observed, config)
    for it in range(config.static_iters):
        loss, lrs = eng.iterate(it)
        if progress is not None:
            progress({"stage": "static", "iteration": it, "loss": loss,
                      "n_balls": eng.B,
                      **{f"lr_{k}": v for k, v in lrs.items()}})
        if (it + 1) % config.prune_every == 0:
            eng.prune()
    return eng.balls()
