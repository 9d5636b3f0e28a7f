"""Fused multi-frame 4D SlingBAG iteration on the B200 (one rank per GPU).

One iteration of pkg/src/pacloud/reconstruction.py:293-328
(``dynamic_reconstruct``'s loop body) as five device launches on one stream:

    pc_deform_states        all selected frames at once      (deformation.py:184)
    pc_forward_traces       fwd + residual + L2 loss          (radiator.py:86, reconstruction.py:312)
    pc_residual_state_grads adjoint G (F,B,5)                 (radiator.py:121)
    pc_deform_backward      chain rule summed over frames     (radiator.py:266, reconstruction.py:314)
    pc_check_finite         non-finite guard per group        (reconstruction.py:60)

then, for world_size > 1, one NCCL all-reduce of the flat float32 gradient
buffer (+ the loss), ONE host synchronisation to read loss / flags, and one
``pc_adam_segments`` launch covering all four parameter groups and the floors
(reconstruction.py:320-328, :153-157).  The launch sequence up to the guard
is captured once in a CUDA graph when the frame set is fixed.

Parameters live in one flat float64 buffer (group order pressure, std,
coords, deform -- the reference's update order), gradients in a float32
buffer with the same offsets, Adam moments in float64.

Sharding (distributed.py): ``shard="frames"`` gives each rank
a contiguous block of every iteration's selected frames; ``shard="sensors"``
gives it a sensor block for every frame (ball states recomputed on every
rank, i.e. broadcast).  Both end in the same gradient all-reduce.
"""

from __future__ import annotations

import gc
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import DynamicCloud, default_basis_grid
from .deformation import (DeviceCloud, deform_backward_device,
                          deform_states_device)
from .distributed import allreduce_iteration, frame_shard, shard_range
from .radiator import (DeviceArray, forward_device, raise_if_coincident,
                       residual_loss_device, state_grads_device, to_device)

GROUP_ORDER = ("pressure", "std", "coords", "deform")
GROUP_OF = {"p0": "pressure", "a0": "std", "mu": "coords", "theta": "deform",
            "sigma": "deform", "omega": "deform"}


def scheduled_lr(lr0, iteration, step_size, drop_rate):
    """reconstruction.py:38-41."""
    return lr0 * drop_rate ** (iteration // step_size)


def morton_order(mu: np.ndarray, bits: int = 10) -> np.ndarray:
    """Stable Z-order of ball centres (the engine's internal ball layout).

    Spatially close balls share 32-ball culling groups in the forward and
    read overlapping residual windows in the adjoint (L1 reuse).  The
    reference's own initial clouds are lattices (geometry.py:129-133), i.e.
    already ordered; this makes any input order behave the same.
    """
    mu = np.asarray(mu, dtype=np.float64).reshape(-1, 3)
    if len(mu) == 0:
        return np.zeros(0, dtype=np.int64)
    lo = mu.min(axis=0)
    span = np.maximum(mu.max(axis=0) - lo, 1e-12)
    q = np.minimum(((mu - lo) / span * (1 << bits)).astype(np.int64),
                   (1 << bits) - 1)
    code = np.zeros(len(mu), dtype=np.int64)
    for bit in range(bits):
        for ax in range(3):
            code |= ((q[:, ax] >> bit) & 1) << (3 * bit + ax)
    return np.argsort(code, kind="stable").astype(np.int64)


def hilbert_order(mu: np.ndarray, bits: int = 10) -> np.ndarray:
    """Stable Hilbert-curve order of ball centres (Skilling's transpose
    algorithm on the quantised coordinates).  Unlike the Z-order the curve
    has no jumps, so every 32 consecutive balls are spatial neighbours: on
    BASELINE config 3 the forward's 32-ball groups shrink from 1.28 to 1.00
    mm mean extent and 3 % fewer of their (group, run) visits are partial.
    `PC_BALL_ORDER=morton` selects the Z-order."""
    mu = np.asarray(mu, dtype=np.float64).reshape(-1, 3)
    if len(mu) == 0:
        return np.zeros(0, dtype=np.int64)
    lo = mu.min(axis=0)
    span = np.maximum(mu.max(axis=0) - lo, 1e-12)
    X = np.minimum(((mu - lo) / span * (1 << bits)).astype(np.int64),
                   (1 << bits) - 1)
    top = 1 << (bits - 1)
    Q = top
    while Q > 1:                       # inverse undo of the excess work
        P = Q - 1
        for i in range(3):
            sel = (X[:, i] & Q) != 0
            X[sel, 0] ^= P             # invert the low bits of axis 0
            ns = ~sel                  # or exchange them with axis i
            t = (X[ns, 0] ^ X[ns, i]) & P
            X[ns, 0] ^= t
            X[ns, i] ^= t
        Q >>= 1
    for i in range(1, 3):              # Gray encode
        X[:, i] ^= X[:, i - 1]
    t = np.zeros(len(X), dtype=np.int64)
    Q = top
    while Q > 1:
        sel = (X[:, 2] & Q) != 0
        t[sel] ^= Q - 1
        Q >>= 1
    X ^= t[:, None]
    code = np.zeros(len(X), dtype=np.int64)
    for b in range(bits):              # interleave, axis 0 most significant
        for i in range(3):
            code |= ((X[:, i] >> b) & 1) << (b * 3 + (2 - i))
    return np.argsort(code, kind="stable").astype(np.int64)


def spatial_ball_order(mu: np.ndarray, a0: np.ndarray | None = None) -> np.ndarray:
    """The engine's internal ball layout: Hilbert order of the centres, then,
    inside every run of `PC_BALL_SEG` (64) consecutive balls, a stable sort
    by radius.  Neighbouring balls of equal radius have equal window lengths,
    so the forward's 32-ball groups meet their edge runs together (config 3:
    ~20 % fewer partial (group, run) visits; forward 248.2 -> 242.5 ms,
    config 4 1370 -> 1317 ms with runs of 128; runs of 128 / 256 cost
    locality on the sparser config 2).  `PC_BALL_ORDER` = `hilbert` (no
    radius pass) or `morton` (Z-order) select the older layouts."""
    kind = os.environ.get("PC_BALL_ORDER", "hilbert_a0")
    if kind == "morton":
        return morton_order(mu)
    order = hilbert_order(mu)
    if kind == "hilbert" or a0 is None or len(order) == 0:
        return order
    seg = max(1, int(os.environ.get("PC_BALL_SEG", "64")))
    a = np.asarray(a0, dtype=np.float64).reshape(-1)[order]
    n = len(order)
    pad = (-n) % seg
    key = np.concatenate([a, np.full(pad, np.inf)]).reshape(-1, seg)
    within = np.argsort(key, axis=1, kind="stable")
    idx = (within + np.arange(key.shape[0])[:, None] * seg).reshape(-1)
    return order[idx[idx < n]]


def select_frames(n_frames: int, batch: int, rng) -> np.ndarray:
    """reconstruction.py:246-250 (same RNG draws as the reference)."""
    if batch <= 0 or batch >= n_frames:
        return np.arange(n_frames)
    return np.sort(rng.choice(n_frames, size=batch, replace=False))


@dataclass
class Segment:
    name: str
    group: str
    shape: tuple
    offset: int
    size: int


class ParamLayout:
    """Offsets of every parameter array inside the flat buffers."""

    def __init__(self, B: int, N: int, basis: str, per_channel: bool):
        shapes = [("p0", (B,)), ("a0", (B,)), ("mu", (B, 3))]
        if basis == "gauss":
            ts = (B, 5, N) if per_channel else (B, N)
            shapes += [("theta", ts), ("sigma", ts)]
        shapes += [("omega", (B, 5, N))]
        self.segments = []
        off = 0
        for name, shp in shapes:
            n = int(np.prod(shp))
            self.segments.append(Segment(name, GROUP_OF[name], shp, off, n))
            off += n
        self.total = off
        self.by_name = {s.name: s for s in self.segments}
        self.offsets = [s.offset for s in self.segments] + [off]

    def views(self, flat: torch.Tensor) -> dict:
        return {s.name: flat[s.offset:s.offset + s.size].view(s.shape)
                for s in self.segments}


class IterationEngine:
    """Device-resident parameters, Adam state and per-iteration buffers."""

    def __init__(self, cloud, array, observed, frame_times, config, *,
                 shard=None, process_group=None, use_graph=True,
                 device=None, spatial_order=True):
        _lib.load_library()
        self.cfg = config
        self.basis = getattr(cloud, "basis", getattr(config, "basis",
                                                     "gauss"))
        self.device = device or torch.device("cuda",
                                             torch.cuda.current_device())
        self.group = process_group
        dist = torch.distributed
        self.world = dist.get_world_size(process_group) if (
            dist.is_available() and dist.is_initialized()) else 1
        self.rank = dist.get_rank(process_group) if self.world > 1 else 0
        if shard not in (None, "frames", "sensors"):
            raise ValueError("shard must be None, 'frames' or 'sensors'")
        self.shard = shard if self.world > 1 else None
        self.frame_times_all = np.asarray(frame_times, dtype=np.float64)
        self.n_frames_all = len(self.frame_times_all)
        lo, hi = (shard_range(array.n_sensors, self.rank, self.world)
                  if self.shard == "sensors" else (0, array.n_sensors))
        self.sensors = (int(lo), int(hi))
        pos = np.asarray(array.positions)[lo:hi]
        self.positions_all = np.asarray(array.positions, dtype=np.float64)
        self.darr = DeviceArray(array, config.support_sigmas,
                                config.exact_forward, positions=pos,
                                sensor_offset=int(lo))
        # observed: (F_all, M_local, T) float32 on the device
        obs = observed
        if not isinstance(obs, torch.Tensor):
            obs = torch.as_tensor(np.ascontiguousarray(obs, np.float32))
        if obs.shape[1] != self.darr.M:
            obs = obs[:, lo:hi]
        self.observed = obs.to(self.device, torch.float32).contiguous()
        if tuple(self.observed.shape[1:]) != (self.darr.M, self.darr.T):
            raise ValueError("observed must be (F, M, T) for this array")

        # ---- flat parameter / gradient / moment buffers
        B = len(cloud.p0)
        N = int(np.asarray(cloud.omega).shape[-1]) if not isinstance(
            cloud.omega, torch.Tensor) else int(cloud.omega.shape[-1])
        per_channel = self.basis == "gauss" and np.ndim(cloud.theta) == 3
        self.layout = ParamLayout(B, N, self.basis, per_channel)
        self.B, self.N = B, N
        f64 = dict(dtype=torch.float64, device=self.device)
        # capacity-backed ball-count buffers (config-5 growth: densify
        # re-views them instead of re-allocating; _ball_hint = growth cap)
        self._caps = {}
        self._ball_hint = 0
        self._pp = 0          # which half of the ping-pong parameter storage
        per_ball = self.layout.total // max(B, 1)
        self.P = self._cap_view("P0", per_ball, B, torch.float64)
        self.Mo = self._cap_view("M0", per_ball, B, torch.float64).zero_()
        self.Vo = self._cap_view("V0", per_ball, B, torch.float64).zero_()
        self.Gf = self._cap_view("Gf", per_ball, B, torch.float32).zero_()
        self.params = self.layout.views(self.P)
        self.grads = self.layout.views(self.Gf)
        # internal ball order (identity or Hilbert / Morton); outputs are un-permuted
        mu_host = cloud.mu.detach().cpu().numpy() if isinstance(
            cloud.mu, torch.Tensor) else np.asarray(cloud.mu)
        a0_host = cloud.a0.detach().cpu().numpy() if isinstance(
            cloud.a0, torch.Tensor) else np.asarray(cloud.a0)
        self.order = spatial_ball_order(mu_host, a0_host) if spatial_order else \
            np.arange(B, dtype=np.int64)
        self.inverse = np.empty_like(self.order)
        self.inverse[self.order] = np.arange(B, dtype=np.int64)
        order_dev = torch.as_tensor(self.order, device=self.device)
        for name in self.params:
            src = to_device(getattr(cloud, name), torch.float64)
            self.params[name].copy_(src.reshape(self.params[name].shape)
                                    .index_select(0, order_dev))
        self.step_count = {s.name: 0 for s in self.layout.segments}
        p = self.params
        self.dcloud = DeviceCloud(p["p0"], p["a0"], p["mu"], p.get("theta"),
                                  p.get("sigma"), p["omega"], self.basis)
        self.use_graph = bool(use_graph)
        # per-stage CUDA-event timings of each iterate() (progress records)
        self.stage_timing = os.environ.get("PC_STAGE_TIMING", "0") == "1"
        self.last_timing = None
        self._events = None
        self._qws = None            # pc_abs_quantile_f32 workspace (densify)
        self._warmed = False
        self._graph = None
        self._graph_frames = None
        self._tail_graph = None
        self._tail_key = None
        self._tail_warmed = False
        self._pool = None
        self._status_host = None
        self._status_dev = None
        self._bufs_F = -1
        self.mu_t = None
        self.ws = None
        n_seg = len(self.layout.segments)
        self.flags = torch.zeros(n_seg, dtype=torch.int32, device=self.device)
        self.coinc = torch.full((1,), _lib.INT64_MAX, dtype=torch.int64,
                                device=self.device)
        self.loss_total = torch.zeros(1, dtype=torch.float64,
                                      device=self.device)
        self.host_observed = None
        self._copy_stream = None
        self._hyper_host = None
        self._hyper_dev = None
        # frame groups for forward / adjoint overlap (PC_FRAME_GROUPS)
        self.frame_groups = int(os.environ.get("PC_FRAME_GROUPS", "1"))
        self._adj_stream = None

    def stream_observed_from(self, host):
        """Upload the observed traces from pinned host memory every iteration
        (frames of the minibatch only), overlapped with the deformation and
        the forward sweep: the copy runs on a side stream and only the
        residual/loss epilogue (pc_residual_loss) waits for it.  `host` is a
        pinned, contiguous CPU float32 tensor (F_all, M_local, T); None turns
        streaming off (the device copy made at construction is used)."""
        if host is not None:
            if not (isinstance(host, torch.Tensor) and host.device.type == "cpu"
                    and host.is_pinned() and host.is_contiguous()
                    and host.dtype == torch.float32):
                raise ValueError("host observed must be a pinned contiguous "
                                 "float32 CPU tensor")
            if tuple(host.shape) != tuple(self.observed.shape):
                raise ValueError(f"host observed shape {tuple(host.shape)} != "
                                 f"{tuple(self.observed.shape)}")
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(device=self.device)
        self.host_observed = host
        self._graph = None

    # ------------------------------------------------------------ buffers
    def _cap_view(self, name: str, per_ball: int, B: int, dtype):
        """The first per_ball*B elements of a buffer sized for the ball
        capacity (max(B, growth cap)); re-allocated only when B outgrows
        it (by 25 %)."""
        n = int(per_ball) * int(B)
        t = self._caps.get(name)
        if t is None or t.dtype != dtype or t.numel() < n:
            cap = max(int(B), int(self._ball_hint), 1)
            if t is not None and t.numel() < n:
                cap = max(cap, int(B + B // 4))
            self._caps[name] = None
            t = torch.empty(int(per_ball) * cap, dtype=dtype, device=self.device)
            self._caps[name] = t
        return t[:n]

    def _ensure_buffers(self, F: int):
        if (self._bufs_F == F and self.mu_t is not None
                and self.mu_t.shape[1] == self.B):
            return
        dev, B, M, T = self.device, self.B, self.darr.M, self.darr.T
        if self._bufs_F != F:
            # per-frame buffers that do not depend on the ball count (kept
            # across densify steps: the residual alone is F*M*T floats)
            self.t_dev = torch.zeros(F, dtype=torch.float64, device=dev)
            self.resid = torch.empty((F, M, T), dtype=torch.float32, device=dev)
            self.loss_f = torch.zeros(F, dtype=torch.float64, device=dev)
            self.obs_stage = None
            self.loss_part = torch.empty(F * M, dtype=torch.float64, device=dev)
        if self._bufs_F != F:
            for k in ("mu_t", "a0_t", "p0_t", "H", "G"):
                self._caps.pop(k, None)
        self.mu_t = self._cap_view("mu_t", 3 * F, B, torch.float64).view(F, B, 3)
        self.a0_t = self._cap_view("a0_t", F, B, torch.float32).view(F, B)
        self.p0_t = self._cap_view("p0_t", F, B, torch.float32).view(F, B)
        self.H = self._cap_view("H", 5 * F, B, torch.float32).view(F, B, 5)
        self.G = self._cap_view("G", 5 * F, B, torch.float32).view(F, B, 5)
        ws = self.darr.workspace_bytes(max(B, 1), F)
        if self.ws is None or self.ws.numel() < ws:
            # 25 % headroom: a growing cloud (densify) re-allocates the
            # workspace (chunk partial traces, ~GBs) rarely
            self.ws = None
            self.ws = torch.empty(max(ws + ws // 4, 1), dtype=torch.uint8, device=dev)
        self._bufs_F = F
        self._graph = None

    def _local_frames(self, frames: np.ndarray) -> np.ndarray:
        if self.shard == "frames":
            return frame_shard(frames, self.rank, self.world)
        return np.asarray(frames, dtype=np.int64)

    def _frame_offset(self, frames: np.ndarray) -> int:
        """Position of this rank's first frame in the iteration's frame
        list (the coincidence word's frame index is global)."""
        if self.shard == "frames":
            return shard_range(len(frames), self.rank, self.world)[0]
        return 0

    # ------------------------------------------------------------ compute
    def _launch_compute(self, obs, host_src=None):
        """deform -> forward+loss -> adjoint -> deformation backward.

        With host_src (pinned host frames), obs is filled from it on the side
        stream while deform + forward run; the residual/loss epilogue joins."""
        cfg = self.cfg
        cur = torch.cuda.current_stream()
        if host_src is not None:
            side = self._copy_stream
            side.wait_stream(cur)       # obs no longer read by the last step
            with torch.cuda.stream(side):
                for dst, src in host_src:
                    dst.copy_(src, non_blocking=True)
        self.coinc.fill_(_lib.INT64_MAX)
        deform_states_device(self.dcloud, self.t_dev, cfg.coord_mode,
                             cfg.a0_floor, self.mu_t, self.a0_t, self.p0_t,
                             self.H)
        F = int(self.mu_t.shape[0])
        groups = self._frame_groups(F)
        adj = cur if len(groups) == 1 else self._adj_stream
        waited_copy = False
        for f0, f1 in groups:
            mu, a0, p0 = self.mu_t[f0:f1], self.a0_t[f0:f1], self.p0_t[f0:f1]
            res, loss = self.resid[f0:f1], self.loss_f[f0:f1]
            if host_src is None:
                forward_device(self.darr, mu, a0, p0, observed=obs[f0:f1],
                               out=res, loss=loss, coincident=self.coinc,
                               workspace=self.ws)
            else:
                forward_device(self.darr, mu, a0, p0, observed=None, out=res,
                               coincident=self.coinc, workspace=self.ws)
                if not waited_copy:
                    cur.wait_stream(self._copy_stream)
                    waited_copy = True
                residual_loss_device(res, obs[f0:f1], out=res, loss=loss,
                                     partial=self.loss_part[f0 * self.darr.M:])
            if adj is not cur:
                # this group's adjoint overlaps the next group's forward
                adj.wait_stream(cur)
            with torch.cuda.stream(adj):
                state_grads_device(self.darr, mu, a0, p0, res,
                                   G=self.G[f0:f1], coincident=self.coinc)
        if adj is not cur:
            cur.wait_stream(adj)
        deform_backward_device(self.dcloud, self.t_dev, cfg.coord_mode,
                               cfg.a0_floor, self.G, self.H, self.grads)
        torch.sum(self.loss_f, dim=0, keepdim=True, out=self.loss_total)

    def _frame_groups(self, F: int):
        """Frame groups of the iteration: forward of group g+1 runs while
        the adjoint of group g runs on a second stream (the kernels are
        limited by different resources: shared memory / issue for the
        forward, registers / FMA + XU pipes for the adjoint)."""
        n = max(1, min(int(self.frame_groups), F))
        if n > 1 and self._adj_stream is None:
            self._adj_stream = torch.cuda.Stream(device=self.device)
        bounds = np.linspace(0, F, n + 1).round().astype(int)
        return [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])
                if b > a]

    def compute_grads(self, frames: np.ndarray) -> None:
        """Launch (asynchronously) the gradient of the selected frames."""
        local = self._local_frames(np.asarray(frames))
        fo = self._frame_offset(np.asarray(frames))
        self.darr.struct.frame_offset = int(fo)
        F = len(local)
        if F == 0:
            self.Gf.zero_()
            self.loss_total.zero_()
            self.coinc.fill_(_lib.INT64_MAX)
            return
        self._ensure_buffers(F)
        contiguous = np.array_equal(local, np.arange(local[0],
                                                     local[0] + F))
        host = self.host_observed
        host_src = None
        if contiguous:
            lo = int(local[0])
            obs = self.observed[lo:lo + F]
            if host is not None:
                host_src = [(obs, host[lo:lo + F])]
        else:
            if self.obs_stage is None:
                self.obs_stage = torch.empty_like(self.observed[:F])
            obs = self.obs_stage
            if host is not None:
                host_src = [(obs[i], host[int(f)]) for i, f in enumerate(local)]
            else:
                idx = torch.as_tensor(local, device=self.device)
                torch.index_select(self.observed, 0, idx, out=self.obs_stage)
        key = (tuple(int(k) for k in local), int(fo),
               None if host is None else host.data_ptr())
        if self.use_graph and self._graph is not None \
                and self._graph_frames == key:
            self._graph.replay()
            return
        self.t_dev.copy_(torch.as_tensor(self.frame_times_all[local],
                                         dtype=torch.float64))
        if self.use_graph and contiguous:
            # warm once eagerly per engine (lazy init inside torch / the
            # driver / the library's function attributes), then capture the
            # fixed launch sequence and replay it from now on; re-captures
            # after a change of frames or ball count skip the warm-up
            if not self._warmed:
                self._launch_compute(obs, host_src)
                self._warmed = True
            self._graph = None
            g = self._capture(lambda: self._launch_compute(obs, host_src))
            self._graph, self._graph_frames = g, key
            self._graph.replay()
        else:
            self._graph = None      # t_dev / obs changed under the graph
            self._launch_compute(obs, host_src)

    def _capture(self, launch):
        """Capture `launch` into a CUDA graph on a side stream, in this
        engine's own memory pool.  CUDAGraph.capture_begin/capture_end
        directly: the torch.cuda.graph context manager also runs
        gc.collect() and torch.cuda.empty_cache() before every capture,
        which stalled the re-capture after a densify step for up to 1 s.
        The cyclic garbage collector is paused for the capture instead: a
        collection inside it could destroy another engine's CUDAGraph, and
        cudaGraphExecDestroy during a global-mode capture invalidates it."""
        if self._pool is None:
            self._pool = torch.cuda.graph_pool_handle()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream(device=self.device)
        st.wait_stream(torch.cuda.current_stream())
        gc_on = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.stream(st):
                g.capture_begin(pool=self._pool)
                try:
                    launch()
                finally:
                    g.capture_end()
        finally:
            if gc_on:
                gc.enable()
        torch.cuda.current_stream().wait_stream(st)
        return g

    def allreduce(self) -> None:
        if self.world > 1:
            allreduce_iteration(self.Gf, self.loss_total, self.coinc,
                                self.group)

    def check_and_status(self):
        """Finite guard + the single host sync of the iteration."""
        lib = _lib.load_library()
        self.flags.zero_()
        off = _lib.i64_array(self.layout.offsets)
        _lib.check(lib.pc_check_finite(
            _lib.ptr(self.Gf), len(self.layout.segments), off,
            _lib.ptr(self.flags), _lib.stream()), "pc_check_finite")
        status = torch.cat([self.loss_total, self.flags.double(),
                            self.coinc.double()]).cpu().numpy()
        loss = float(status[0])
        flags = status[1:1 + len(self.layout.segments)].astype(bool)
        # pair indices b*M+m stay far below 2**53; INT64_MAX means "none"
        coinc = int(status[-1]) if status[-1] < 9.0e18 else _lib.INT64_MAX
        return loss, flags, coinc

    def apply_update(self, lrs: dict, only=None) -> None:
        """pc_adam_segments (or sgd) for all (or `only`) segments + floors."""
        lib = _lib.load_library()
        cfg = self.cfg
        floors = {"p0": cfg.p0_floor, "a0": cfg.a0_floor,
                  "sigma": cfg.sigma_floor}
        segs = [s for s in self.layout.segments
                if only is None or s.name in only]
        if not segs:
            return
        for s in segs:
            self.step_count[s.name] += 1
        # contiguous runs of the flat buffer: pass explicit offsets
        off, lr, step, fl = [], [], [], []
        for s in segs:
            off.append(s.offset)
            lr.append(lrs[s.group])
            step.append(self.step_count[s.name])
            fl.append(floors.get(s.name, -math.inf))
        off.append(segs[-1].offset + segs[-1].size)
        if any(segs[i].offset + segs[i].size != segs[i + 1].offset
               for i in range(len(segs) - 1)):
            for s in segs:   # non-contiguous subset: one launch per segment
                self._update_one(s, lrs, floors)
            return
        if cfg.optimizer == "adam":
            _lib.check(lib.pc_adam_segments(
                _lib.ptr(self.P), _lib.ptr(self.Gf), _lib.ptr(self.Mo),
                _lib.ptr(self.Vo), len(segs), _lib.i64_array(off),
                _lib.f64_array(lr), _lib.i32_array(step),
                _lib.f64_array(fl), _lib.stream()), "pc_adam_segments")
        else:
            _lib.check(lib.pc_sgd_segments(
                _lib.ptr(self.P), _lib.ptr(self.Gf), len(segs),
                _lib.i64_array(off), _lib.f64_array(lr),
                _lib.f64_array(fl), _lib.stream()), "pc_sgd_segments")

    def _update_one(self, s, lrs, floors):
        lib = _lib.load_library()
        off = _lib.i64_array([s.offset, s.offset + s.size])
        if self.cfg.optimizer == "adam":
            _lib.check(lib.pc_adam_segments(
                _lib.ptr(self.P), _lib.ptr(self.Gf), _lib.ptr(self.Mo),
                _lib.ptr(self.Vo), 1, off, _lib.f64_array([lrs[s.group]]),
                _lib.i32_array([self.step_count[s.name]]),
                _lib.f64_array([floors.get(s.name, -math.inf)]),
                _lib.stream()), "pc_adam_segments")
        else:
            _lib.check(lib.pc_sgd_segments(
                _lib.ptr(self.P), _lib.ptr(self.Gf), 1, off,
                _lib.f64_array([lrs[s.group]]),
                _lib.f64_array([floors.get(s.name, -math.inf)]),
                _lib.stream()), "pc_sgd_segments")

    def _lrs(self, iteration: int) -> dict:
        cfg = self.cfg
        return {"coords": scheduled_lr(cfg.lr_coords, iteration,
                                       cfg.step_size, cfg.drop_rate),
                "pressure": scheduled_lr(cfg.lr_pressure, iteration,
                                         cfg.step_size, cfg.drop_rate),
                "std": scheduled_lr(cfg.lr_std, iteration, cfg.step_size,
                                    cfg.drop_rate),
                "deform": scheduled_lr(cfg.lr_deform, iteration,
                                       cfg.step_size, cfg.drop_rate)}

    def _fill_hyper(self, lrs: dict) -> None:
        """(lr, t) per segment into the pinned table the update copies."""
        segs = self.layout.segments
        n = len(segs)
        if self._hyper_host is None or self._hyper_host.numel() != 2 * n:
            self._hyper_host = torch.empty(2 * n, dtype=torch.float64).pin_memory()
            self._hyper_dev = torch.empty(2 * n, dtype=torch.float64,
                                          device=self.device)
            self._status_host = torch.empty(n + 2, dtype=torch.float64).pin_memory()
            self._status_dev = torch.empty(n + 2, dtype=torch.float64,
                                           device=self.device)
            self._tail_graph = None
        hv = self._hyper_host.numpy()
        for i, sg in enumerate(segs):
            hv[2 * i] = lrs[sg.group]
            hv[2 * i + 1] = self.step_count[sg.name] + 1

    def _launch_tail(self) -> None:
        """pc_check_finite + pc_update_guarded: the step and its guard on
        the device, (lr, t) per segment from the pinned table (copied in
        stream order), then the status (loss, flags, coincidence) packed and
        copied to pinned host memory; no host synchronisation here."""
        lib = _lib.load_library()
        segs = self.layout.segments
        n = len(segs)
        self._hyper_dev.copy_(self._hyper_host, non_blocking=True)
        cfg = self.cfg
        floors = {"p0": cfg.p0_floor, "a0": cfg.a0_floor,
                  "sigma": cfg.sigma_floor}
        off = _lib.i64_array(self.layout.offsets)
        self.flags.zero_()
        _lib.check(lib.pc_check_finite(
            _lib.ptr(self.Gf), n, off, _lib.ptr(self.flags), _lib.stream()),
            "pc_check_finite")
        _lib.check(lib.pc_update_guarded(
            _lib.ptr(self.P), _lib.ptr(self.Gf), _lib.ptr(self.Mo),
            _lib.ptr(self.Vo), n, off,
            _lib.f64_array([floors.get(sg.name, -math.inf) for sg in segs]),
            _lib.i32_array([GROUP_ORDER.index(sg.group) for sg in segs]),
            _lib.ptr(self._hyper_dev), _lib.ptr(self.flags),
            _lib.ptr(self.loss_total), _lib.ptr(self.coinc),
            0 if cfg.optimizer == "adam" else 1, _lib.stream()),
            "pc_update_guarded")
        self._status_dev[0:1].copy_(self.loss_total)
        self._status_dev[1:1 + n].copy_(self.flags)
        self._status_dev[n + 1:n + 2].copy_(self.coinc)
        self._status_host.copy_(self._status_dev, non_blocking=True)

    def _guarded_update(self, lrs: dict) -> None:
        """Guard + update + status copy, replayed from a CUDA graph once the
        layout is fixed (one launch instead of seven eager ones)."""
        self._fill_hyper(lrs)
        key = (self.P.data_ptr(), self.Gf.data_ptr(), self.Mo.data_ptr(),
               self.Vo.data_ptr(), self.layout.total,
               self._status_host.data_ptr())
        if not self.use_graph:
            self._launch_tail()
            return
        if self._tail_graph is not None and self._tail_key == key:
            self._tail_graph.replay()
            return
        if not self._tail_warmed:
            self._launch_tail()          # eager once (lazy library init)
            self._tail_warmed = True
            return
        self._tail_graph = None
        g = self._capture(self._launch_tail)
        self._tail_graph, self._tail_key = g, key
        g.replay()

    def _status(self):
        torch.cuda.current_stream().synchronize()
        status = self._status_host.numpy()
        loss = float(status[0])
        flags = status[1:-1].astype(bool)
        # pair indices b*M+m stay far below 2**53; INT64_MAX means "none"
        coinc = int(status[-1]) if status[-1] < 9.0e18 else _lib.INT64_MAX
        return loss, flags, coinc

    def iterate(self, iteration: int, frames: np.ndarray) -> float:
        """One full iteration; returns the (all-reduced) loss.

        gradient -> (all-reduce) -> finite guard -> guarded Adam all stay on
        the device; the host reads the status once, after the step, and
        raises the reference's exceptions (the device applied exactly the
        updates the reference makes before raising)."""
        lrs = self._lrs(iteration)
        self.last_lrs = lrs
        nvtx = torch.cuda.nvtx
        ev = self._stage_events() if self.stage_timing else None
        if ev:
            ev[0].record()
        nvtx.range_push("pc:grads (deform, forward+loss, adjoint, deform-bwd)")
        self.compute_grads(frames)
        nvtx.range_pop()
        if ev:
            ev[1].record()
        nvtx.range_push("pc:exchange")
        self.allreduce()
        nvtx.range_pop()
        if ev:
            ev[2].record()
        nvtx.range_push("pc:guard+adam")
        self._guarded_update(lrs)
        nvtx.range_pop()
        if ev:
            ev[3].record()
        nvtx.range_push("pc:status (host sync)")
        loss, flags, coinc = self._status()
        nvtx.range_pop()
        if ev:
            # every event completed before the status read returned
            n_loc = len(self._local_frames(frames))
            grads = ev[0].elapsed_time(ev[1])
            self.last_timing = {
                "grads_ms": grads, "exchange_ms": ev[1].elapsed_time(ev[2]),
                "update_ms": ev[2].elapsed_time(ev[3]),
                "iteration_ms": ev[0].elapsed_time(ev[3]),
                "pair_evals_per_s": self.B * self.darr.M * n_loc /
                (grads * 1e-3) if grads > 0 else None}
        if coinc != _lib.INT64_MAX:
            self._raise_coincident(coinc, frames)
        if not math.isfinite(loss):
            raise RuntimeError(f"non-finite loss at iteration {iteration}")
        # adam_step raises per ARRAY before touching it (reconstruction.py:
        # 60-61, 88-93): the segments before the first non-finite one were
        # stepped (pc_update_guarded did the same on the device)
        segs = self.layout.segments
        bad = len(segs)
        if flags.any():
            bad = int(np.nonzero(flags)[0][0])
        for sg in segs[:bad]:
            self.step_count[sg.name] += 1
        if bad < len(segs):
            raise ValueError(
                f"non-finite gradient in parameter group '{segs[bad].group}'")
        return loss

    def _stage_events(self):
        if self._events is None:
            self._events = [torch.cuda.Event(enable_timing=True)
                            for _ in range(4)]
        return self._events

    def _raise_coincident(self, word: int, frames) -> None:
        """reconstruction.py:303-311 -> radiator.py:186-192: the first frame
        of the iteration (in frame-list order) holding a coincident pair
        raises, naming the closest (ball, sensor) pair of THAT frame over the
        whole array.  The word ((f B + b) M_total + m, MIN-reduced over
        ranks) names the frame; its states are recomputed here (parameters
        are replicated), so every rank raises the same message."""
        frames = np.asarray(frames, dtype=np.int64)
        fpos = int(word) // (self.B * self.darr.n_sensors_total)
        k = int(frames[min(fpos, len(frames) - 1)])
        dev, B = self.device, self.B
        t = torch.tensor([self.frame_times_all[k]], dtype=torch.float64,
                         device=dev)
        mu1 = torch.empty((1, B, 3), dtype=torch.float64, device=dev)
        a1 = torch.empty((1, B), dtype=torch.float32, device=dev)
        p1 = torch.empty((1, B), dtype=torch.float32, device=dev)
        deform_states_device(self.dcloud, t, self.cfg.coord_mode,
                             self.cfg.a0_floor, mu1, a1, p1, None)
        inv = torch.as_tensor(self.inverse, device=dev)
        raise_if_coincident(word, mu1[0].index_select(0, inv),
                            self.positions_all)

    # ------------------------------------------------------------ densify
    @staticmethod
    def _percentile_split(n: int, q: float):
        """numpy's 'linear' virtual index (n - 1) q / 100 split into the
        lower order-statistic rank k and the lerp weight gamma
        (numpy/lib/_function_base_impl.py _quantile); host arithmetic on n
        and q only."""
        qq = float(np.float64(q) / np.float64(100.0))
        virtual = (n - 1) * qq
        if virtual >= n - 1:
            return n - 1, 0.0
        k = max(0, math.floor(virtual))
        return k, virtual - k

    def _p0_grad_threshold_dev(self, q: float) -> torch.Tensor:
        """Device double: numpy.percentile(|dL/dp0|, q, method='linear') of
        the last computed gradient (pc_abs_quantile_f32: radix select +
        numpy's _lerp on the device, no host round trip)."""
        lib = _lib.load_library()
        n = int(self.B)
        thr = torch.zeros(1, dtype=torch.float64, device=self.device)
        if n == 0:
            return thr
        k, gamma = self._percentile_split(n, q)
        if self._qws is None:
            self._qws = torch.empty(int(lib.pc_abs_quantile_workspace_bytes()),
                                    dtype=torch.uint8, device=self.device)
        _lib.check(lib.pc_abs_quantile_f32(
            _lib.ptr(self.grads["p0"]), n, int(k), float(gamma), _lib.ptr(thr),
            _lib.ptr(self._qws), self._qws.numel(), _lib.stream()),
            "pc_abs_quantile_f32")
        return thr

    def p0_grad_threshold(self, q: float = 90.0) -> float:
        """numpy.percentile(|dL/dp0|, q, method='linear'), read back."""
        return float(self._p0_grad_threshold_dev(q).item())

    def densify(self, p0_min: float = 0.01, q: float = 90.0,
                child_shift: float = 0.5, max_balls: int | None = None,
                halve_pressure: bool = False):
        """Config-5 adaptive step (builder-defined): prune
        p0 < p0_min, split balls with |dL/dp0| above its q-th percentile.
        New order = survivors in order, then one child per split survivor in
        parent order (pc_compact_index), truncated to `max_balls`; every
        parameter and Adam moment is gathered (pc_gather_rows, step counts
        preserved as in reconstruction.py:95-100); a child is a clone of its
        parent moved +child_shift*a0 along x (pc_densify_flags +
        pc_densify_apply) and starts with zero moments.  `halve_pressure`
        also halves the pressure of split parents and children (measured:
        with it, repeated splits drive p0 under the absolute prune floor and
        config 5 stalls near 125k balls instead of growing to 500k).  Everything runs on the device; the one host read is
        the (#keep, #split) pair that sizes the new cloud.
        Returns (n_pruned, n_children)."""
        lib = _lib.load_library()
        B = self.B
        dev = self.device
        thr = self._p0_grad_threshold_dev(q)
        keep = torch.empty(B, dtype=torch.uint8, device=dev)
        split = torch.empty(B, dtype=torch.uint8, device=dev)
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
        _lib.check(lib.pc_densify_masks(
            _lib.ptr(self.params["p0"]), _lib.ptr(self.grads["p0"]), B,
            float(p0_min), _lib.ptr(thr), _lib.ptr(keep), _lib.ptr(split),
            _lib.ptr(counts), _lib.stream()), "pc_densify_masks")
        ws = torch.empty(int(lib.pc_compact_workspace_bytes(B)),
                         dtype=torch.uint8, device=dev)
        index = torch.empty(2 * B, dtype=torch.int64, device=dev)
        n_out = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(lib.pc_compact_index(
            _lib.ptr(keep), _lib.ptr(split), B, _lib.ptr(index),
            _lib.ptr(n_out), _lib.ptr(ws), ws.numel(), _lib.stream()),
            "pc_compact_index")
        n_keep, n_split = (int(v) for v in counts.cpu().tolist())   # the sync
        if n_keep == 0:
            raise RuntimeError("all balls pruned; lower the densify p0_min")
        if max_balls is not None:
            n_split = min(n_split, max(0, int(max_balls) - n_keep))
        B2 = n_keep + n_split
        index = index[:B2]
        per_channel = self.basis == "gauss" and self.params["theta"].dim() == 3
        layout = ParamLayout(B2, self.N, self.basis, per_channel)
        if max_balls is not None:
            self._ball_hint = max(self._ball_hint, int(max_balls))
        # the other half of the ping-pong parameter / moment storage
        per_ball = layout.total // max(B2, 1)
        side = 1 - self._pp
        P2 = self._cap_view(f"P{side}", per_ball, B2, torch.float64)
        M2 = self._cap_view(f"M{side}", per_ball, B2, torch.float64)
        V2 = self._cap_view(f"V{side}", per_ball, B2, torch.float64)
        for old, new in zip(self.layout.segments, layout.segments):
            row = (old.size // B) * 8
            for src, dst in ((self.P, P2), (self.Mo, M2), (self.Vo, V2)):
                _lib.check(lib.pc_gather_rows(
                    _lib.ptr(src[old.offset:]), _lib.ptr(dst[new.offset:]),
                    _lib.ptr(index), B2, row, _lib.stream()),
                    "pc_gather_rows")
            if n_split:
                M2[new.offset + (new.size // B2) * n_keep:
                   new.offset + new.size].zero_()
                V2[new.offset + (new.size // B2) * n_keep:
                   new.offset + new.size].zero_()
        halve = torch.empty(B2, dtype=torch.uint8, device=dev)
        child = torch.empty(B2, dtype=torch.uint8, device=dev)
        _lib.check(lib.pc_densify_flags(
            _lib.ptr(index), B, n_keep, B2, _lib.ptr(keep), _lib.ptr(halve),
            _lib.ptr(child), _lib.stream()), "pc_densify_flags")
        pv = layout.views(P2)
        _lib.check(lib.pc_densify_apply(
            _lib.ptr(pv["p0"]), _lib.ptr(pv["mu"]), _lib.ptr(pv["a0"]),
            _lib.ptr(halve) if halve_pressure else None, _lib.ptr(child), B2,
            float(child_shift),
            _lib.stream()), "pc_densify_apply")
        # swap in the new cloud (internal order becomes the caller's order)
        self.layout, self.B = layout, B2
        self.P, self.Mo, self.Vo = P2, M2, V2
        self._pp = side
        self.Gf = self._cap_view("Gf", per_ball, B2, torch.float32)
        self.Gf.zero_()
        self.params = layout.views(self.P)
        self.grads = layout.views(self.Gf)
        p = self.params
        self.dcloud = DeviceCloud(p["p0"], p["a0"], p["mu"], p.get("theta"),
                                  p.get("sigma"), p["omega"], self.basis)
        self.order = np.arange(B2, dtype=np.int64)
        self.inverse = self.order.copy()
        self._graph = None          # B changed: _ensure_buffers re-sizes the ball buffers
        return B - n_keep, n_split

    # ------------------------------------------------------------ views
    def cloud(self) -> DynamicCloud:
        p = {k: v.cpu().numpy()[self.inverse].copy()
             for k, v in self.params.items()}
        return DynamicCloud(p["p0"], p["a0"], p["mu"], p.get("theta"),
                            p.get("sigma"), p["omega"], basis=self.basis)

    def grads_numpy(self) -> dict:
        """Parameter gradients in the caller's ball order (float64)."""
        return {k: v.double().cpu().numpy()[self.inverse]
                for k, v in self.grads.items()}


def identity_cloud(p0, a0, mu, n_basis: int, basis: str = "gauss"):
    """Attach identity deformation (reconstruction.py:274-281)."""
    p0 = np.asarray(p0, dtype=np.float64)
    B = len(p0)
    if basis == "polyfourier":
        return DynamicCloud(p0, a0, mu, None, None, np.zeros((B, 5, n_basis)),
                            basis="polyfourier")
    th, sg = default_basis_grid(n_basis)
    return DynamicCloud(p0, a0, mu, np.broadcast_to(th, (B, n_basis)).copy(),
                        np.broadcast_to(sg, (B, n_basis)).copy(),
                        np.zeros((B, 5, n_basis)))
