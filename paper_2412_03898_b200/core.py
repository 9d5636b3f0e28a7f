"""Hot-path domain types, mirroring the reference's names and fields.

Mirrors (pkg/src/pacloud): ``Box`` (core.py:35-70), ``GaussBall``
(core.py:74-101), ``VoxelGrid``
(core.py:418-446), ``SensorArray`` (core.py:295-354), ``SignalSet``
(core.py:366-414), ``DynamicCloud`` (core.py:166-259), ``ReconConfig``
(core.py:448-502), ``frame_times`` (core.py:357-363),
``default_basis_grid`` (core.py:152-163), ``CloudState`` /
``BallStateAtT`` / ``CloudStateGrad`` (deformation.py:22-54, 207-216),
``CloudGrads`` (radiator.py:245-263) and ``AdamState``
(reconstruction.py:44-54).  The functions of this package are duck-typed:
the reference's own objects work as inputs too.

Additions for the BASELINE configs: ``DynamicCloud.basis`` selects the
reference Gaussian basis ("gauss") or the cubic-polynomial + Fourier basis
("polyfourier", builder-defined).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

CHANNELS = ("a0", "p0", "mu_x", "mu_y", "mu_z")
N_CHANNELS = 5
COORD_MODES = ("multiplicative", "additive", "radial")
BASES = ("gauss", "polyfourier")


def _vec3(v, what: str) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (3,):
        raise ValueError(f"{what} must be a 3-vector")
    return a


@dataclass(frozen=True)
class Box:
    """Axis-aligned box [lo, hi] in mm (regions of interest, phantoms)."""

    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo, hi = _vec3(self.lo, "lo"), _vec3(self.hi, "hi")
        if (hi < lo).any():
            raise ValueError("box hi must be >= lo on every axis")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    @classmethod
    def cube(cls, half_extent: float, center=(0.0, 0.0, 0.0)) -> "Box":
        c = _vec3(center, "center")
        return cls(c - float(half_extent), c + float(half_extent))

    @property
    def center(self) -> np.ndarray:
        return 0.5 * (self.lo + self.hi)

    @property
    def size(self) -> np.ndarray:
        return self.hi - self.lo

    def corners(self) -> np.ndarray:
        bits = (np.arange(8)[:, None] >> np.arange(3)[None, :]) & 1
        return np.where(bits == 0, self.lo, self.hi)

    def circumradius(self, about=(0.0, 0.0, 0.0)) -> float:
        """Largest distance from `about` to a corner."""
        d = self.corners() - _vec3(about, "about")
        return float(np.sqrt((d * d).sum(axis=1)).max())

    def contains(self, points) -> np.ndarray:
        """Inclusive test for (n, 3) points."""
        p = np.atleast_2d(np.asarray(points, dtype=np.float64))
        return ((p >= self.lo) & (p <= self.hi)).all(axis=1)


@dataclass(frozen=True)
class VoxelGrid:
    """Regular scalar field; `origin` is the centre of voxel (0, 0, 0)."""

    origin: np.ndarray
    spacing: float
    dims: tuple
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "origin", _vec3(self.origin, "origin"))
        object.__setattr__(self, "spacing", float(self.spacing))
        dims = tuple(int(d) for d in self.dims)
        object.__setattr__(self, "dims", dims)
        if not self.spacing > 0:
            raise ValueError("spacing must be > 0")
        if len(dims) != 3 or min(dims) < 1:
            raise ValueError("dims must be three integers >= 1")
        vals = np.ascontiguousarray(self.values, dtype=np.float64)
        if vals.shape != dims:
            if vals.size != int(np.prod(dims)):
                raise ValueError(f"values size {vals.size} != prod(dims) "
                                 f"{int(np.prod(dims))}")
            vals = vals.reshape(dims)
        object.__setattr__(self, "values", vals)

    def voxel_centers_1d(self, axis: int) -> np.ndarray:
        return self.origin[axis] + self.spacing * np.arange(self.dims[axis])


@dataclass(frozen=True)
class GaussBall:
    """One spherical Gaussian source (reference core.py:74-101)."""

    p0: float
    a0: float
    mu: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "p0", float(self.p0))
        object.__setattr__(self, "a0", float(self.a0))
        object.__setattr__(self, "mu", _vec3(self.mu, "mu"))
        if not self.a0 > 0:
            raise ValueError(f"a0 must be > 0, got {self.a0}")
        if self.p0 < 0:
            raise ValueError(f"p0 must be >= 0, got {self.p0}")
        if not (np.isfinite(self.p0) and np.isfinite(self.a0)
                and np.isfinite(self.mu).all()):
            raise ValueError("ball attributes must be finite")


@dataclass(frozen=True)
class DeformField:
    """Gaussian-basis temporal deformation curves for one ball (reference
    core.py:105-135): theta / sigma shared (N,) or per-channel (5, N),
    omega (5, N)."""

    theta: np.ndarray
    sigma: np.ndarray
    omega: np.ndarray

    def __post_init__(self):
        theta = np.asarray(self.theta, dtype=np.float64)
        sigma = np.asarray(self.sigma, dtype=np.float64)
        omega = np.asarray(self.omega, dtype=np.float64)
        if theta.ndim not in (1, 2) or theta.shape != sigma.shape:
            raise ValueError("theta and sigma must share shape (N,) or (5, N)")
        if theta.ndim == 2 and theta.shape[0] != N_CHANNELS:
            raise ValueError(f"per-channel theta must have {N_CHANNELS} rows")
        n = theta.shape[-1]
        if omega.shape != (N_CHANNELS, n):
            raise ValueError(
                f"omega must have shape ({N_CHANNELS}, {n}), got {omega.shape}")
        if np.any(sigma <= 0):
            raise ValueError("all basis widths sigma must be > 0")
        object.__setattr__(self, "theta", theta)
        object.__setattr__(self, "sigma", sigma)
        object.__setattr__(self, "omega", omega)

    @property
    def n_basis(self) -> int:
        return int(self.theta.shape[-1])

    @property
    def shared_basis(self) -> bool:
        return self.theta.ndim == 1

    @classmethod
    def identity(cls, n_basis: int) -> "DeformField":
        """Zero weights over the default theta grid: H(t) = 0 everywhere
        (reference core.py:145-149)."""
        theta, sigma = default_basis_grid(n_basis)
        return cls(theta, sigma, np.zeros((N_CHANNELS, n_basis)))


@dataclass(frozen=True)
class Violation:
    """One invariant violation found by `validate_cloud` (core.py:262-268)."""

    index: int
    field: str
    message: str


def validate_cloud(cloud, roi) -> list:
    """Diagnostic scan of a cloud against the type invariants and an ROI
    (reference core.py:271-292): a0 > 0, p0 >= 0, basis widths > 0, centres
    inside `roi` (inclusive).  Never raises.  Host-side bookkeeping over the
    caller's arrays, as in the reference."""
    out = []
    p0 = np.asarray(cloud.p0, dtype=np.float64)
    a0 = np.asarray(cloud.a0, dtype=np.float64)
    mu = np.asarray(cloud.mu, dtype=np.float64).reshape(-1, 3)
    sigma = getattr(cloud, "sigma", None)
    sigma = None if sigma is None else np.asarray(sigma, dtype=np.float64)
    n = len(p0)
    inside = roi.contains(mu) if n else np.zeros(0, bool)
    for i in range(n):
        if not a0[i] > 0:
            out.append(Violation(i, "a0", f"a0 = {a0[i]} is not > 0"))
        if p0[i] < 0:
            out.append(Violation(i, "p0", f"p0 = {p0[i]} is negative"))
        if sigma is not None and np.any(sigma[i] <= 0):
            out.append(Violation(i, "sigma", "basis width <= 0"))
        if not inside[i]:
            out.append(Violation(
                i, "mu", f"center {mu[i]} outside roi [{roi.lo}, {roi.hi}]"))
    return out


@dataclass(frozen=True)
class SensorArray:
    """Detector positions plus acoustic and sampling parameters."""

    positions: np.ndarray
    sound_speed: float = 1.5
    sample_rate: float = 10.0
    n_samples: int = 2
    t_start: float = 0.0
    radius: float | None = None

    def __post_init__(self):
        pos = np.ascontiguousarray(self.positions, dtype=np.float64)
        if pos.ndim != 2 or pos.shape[1] != 3 or pos.shape[0] < 1:
            raise ValueError(f"positions must be (M, 3), got {pos.shape}")
        object.__setattr__(self, "positions", pos)
        if not self.sound_speed > 0:
            raise ValueError("sound_speed must be > 0")
        if not self.sample_rate > 0:
            raise ValueError("sample_rate must be > 0")
        if self.n_samples < 2:
            raise ValueError("n_samples must be >= 2")

    @property
    def n_sensors(self) -> int:
        return self.positions.shape[0]

    @property
    def dt(self) -> float:
        return 1.0 / self.sample_rate

    def sample_times(self) -> np.ndarray:
        return self.t_start + np.arange(self.n_samples) / self.sample_rate

    def with_window(self, t_start: float, n_samples: int) -> "SensorArray":
        return SensorArray(self.positions, self.sound_speed, self.sample_rate,
                           n_samples, t_start, self.radius)

    def subset(self, lo: int, hi: int) -> "SensorArray":
        """Sensors [lo, hi) -- the shard of a sensor-sharded rank."""
        return SensorArray(self.positions[lo:hi], self.sound_speed,
                           self.sample_rate, self.n_samples, self.t_start,
                           None)


def frame_times(n_frames: int) -> np.ndarray:
    """Normalised frame timestamps t_k = k/(K-1); [0.0] for one frame."""
    if n_frames < 1:
        raise ValueError("n_frames must be >= 1")
    if n_frames == 1:
        return np.zeros(1)
    return np.arange(n_frames, dtype=np.float64) / (n_frames - 1)


def default_basis_grid(n_basis: int):
    """Evenly spaced Gaussian centres on [0, 1], widths of two spacings."""
    if n_basis < 1:
        raise ValueError("n_basis must be >= 1")
    if n_basis == 1:
        return np.array([0.5]), np.array([1.0])
    theta = np.arange(n_basis, dtype=np.float64) / (n_basis - 1)
    return theta, np.full(n_basis, 2.0 / (n_basis - 1))


@dataclass(frozen=True)
class SignalSet:
    """Per-sensor, per-frame traces data[m, k, j] (reference layout)."""

    data: np.ndarray
    frame_times: np.ndarray

    def __post_init__(self):
        data = np.asarray(self.data)
        ft = np.ascontiguousarray(self.frame_times, dtype=np.float64)
        if data.ndim != 3:
            raise ValueError(f"data must be (M, K, T), got shape {data.shape}")
        if ft.shape != (data.shape[1],):
            raise ValueError("frame_times length must equal the frame axis")
        object.__setattr__(self, "frame_times", ft)

    @property
    def n_sensors(self) -> int:
        return self.data.shape[0]

    @property
    def n_frames(self) -> int:
        return self.data.shape[1]

    @property
    def n_samples(self) -> int:
        return self.data.shape[2]

    def frame(self, k: int) -> np.ndarray:
        return self.data[:, k, :]

    def validate_against(self, array) -> None:
        if (self.n_sensors != array.n_sensors
                or self.n_samples != array.n_samples):
            raise ValueError(
                f"signal tensor ({self.n_sensors} sensors x {self.n_samples} "
                f"samples) does not match the array ({array.n_sensors} x "
                f"{array.n_samples})")


@dataclass(frozen=True)
class BallStateAtT:
    a0_t: float
    p0_t: float
    mu_t: np.ndarray


@dataclass(frozen=True)
class CloudState:
    """Instantaneous attributes of a cloud (structure of arrays)."""

    a0_t: np.ndarray
    p0_t: np.ndarray
    mu_t: np.ndarray

    def __post_init__(self):
        b = self.a0_t.shape[0]
        if tuple(self.p0_t.shape) != (b,) or tuple(self.mu_t.shape) != (b, 3):
            raise ValueError("inconsistent cloud state shapes")

    def __len__(self) -> int:
        return self.a0_t.shape[0]

    @classmethod
    def from_states(cls, states) -> "CloudState":
        states = list(states)
        if not states:
            return cls(np.zeros(0), np.zeros(0), np.zeros((0, 3)))
        return cls(np.array([s.a0_t for s in states]),
                   np.array([s.p0_t for s in states]),
                   np.array([s.mu_t for s in states]))


@dataclass(frozen=True)
class CloudStateGrad:
    d_base: np.ndarray
    d_omega: np.ndarray
    d_theta: np.ndarray
    d_sigma: np.ndarray
    omega_row: np.ndarray
    shared_basis: bool


@dataclass
class CloudGrads:
    p0: np.ndarray
    a0: np.ndarray
    mu: np.ndarray
    theta: np.ndarray
    sigma: np.ndarray
    omega: np.ndarray

    def __iadd__(self, other: "CloudGrads") -> "CloudGrads":
        for k in ("p0", "a0", "mu", "theta", "sigma", "omega"):
            setattr(self, k, getattr(self, k) + getattr(other, k))
        return self


class DynamicCloud:
    """Balls with per-ball deformation fields (packed arrays)."""

    def __init__(self, p0, a0, mu, theta, sigma, omega, basis="gauss"):
        if basis not in BASES:
            raise ValueError(f"basis must be one of {BASES}")
        self.basis = basis
        self.p0 = np.ascontiguousarray(p0, dtype=np.float64)
        self.a0 = np.ascontiguousarray(a0, dtype=np.float64)
        self.mu = np.ascontiguousarray(mu, dtype=np.float64)
        self.omega = np.ascontiguousarray(omega, dtype=np.float64)
        b = self.p0.shape[0]
        if basis == "polyfourier":
            self.theta = np.zeros((b, 0))
            self.sigma = np.zeros((b, 0))
        else:
            self.theta = np.ascontiguousarray(theta, dtype=np.float64)
            self.sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        if self.a0.shape != (b,) or self.mu.shape != (b, 3):
            raise ValueError("p0 (B,), a0 (B,) and mu (B, 3) must align")
        n = self.omega.shape[-1]
        if self.omega.shape != (b, N_CHANNELS, n):
            raise ValueError(
                f"omega must be (B, {N_CHANNELS}, N), got {self.omega.shape}")
        if basis == "gauss":
            if self.theta.shape != self.sigma.shape:
                raise ValueError("theta and sigma must share a shape")
            if self.theta.shape not in ((b, n), (b, N_CHANNELS, n)):
                raise ValueError("theta must be (B, N) or (B, 5, N)")
        elif n < 4 or (n - 4) % 2:
            raise ValueError("poly+Fourier basis needs N = 4 + 2*harmonics")

    def __len__(self) -> int:
        return self.p0.shape[0]

    @property
    def n_basis(self) -> int:
        return self.omega.shape[-1]

    @property
    def shared_basis(self) -> bool:
        return self.basis != "gauss" or self.theta.ndim == 2

    @property
    def balls(self) -> list:
        """Baseline attributes as GaussBall records (reference core.py:213)."""
        return [GaussBall(self.p0[i], self.a0[i], self.mu[i])
                for i in range(len(self))]

    @classmethod
    def static(cls, p0, a0, mu, n_basis: int = 1, basis="gauss"):
        """Identity deformation attached to baseline arrays."""
        p0 = np.asarray(p0, dtype=np.float64)
        b = p0.shape[0]
        if basis == "polyfourier":
            return cls(p0, a0, mu, None, None, np.zeros((b, 5, n_basis)),
                       basis="polyfourier")
        th, sg = default_basis_grid(n_basis)
        return cls(p0, a0, mu, np.broadcast_to(th, (b, n_basis)).copy(),
                   np.broadcast_to(sg, (b, n_basis)).copy(),
                   np.zeros((b, N_CHANNELS, n_basis)))


@dataclass(frozen=True)
class ReconConfig:
    """Reconstruction knobs (defaults = the reference's published setup)."""

    lr_coords: float = 5e-7
    lr_pressure: float = 5e-4
    lr_std: float = 5e-7
    lr_deform: float = 5e-6
    step_size: int = 160
    drop_rate: float = 0.1
    static_iters: int = 480
    dynamic_iters: int = 480
    prune_threshold: float = 1e-3
    prune_every: int = 40
    n_basis: int = 65
    a0_floor: float = 0.05
    sigma_floor: float = 1e-4
    p0_floor: float = 0.0
    init_pitch: float = 2.0
    init_p0_scale: float = 1e-3
    coord_mode: str = "multiplicative"
    optimizer: str = "adam"
    frame_batch: int = 0
    reference_frame: int = 0
    support_sigmas: float = 6.0
    exact_forward: bool = False
    seed: int = 0
    basis: str = "gauss"

    def __post_init__(self):
        for name in ("lr_coords", "lr_pressure", "lr_std", "lr_deform"):
            if not getattr(self, name) > 0:
                raise ValueError(f"{name} must be > 0")
        if not 0 < self.drop_rate <= 1:
            raise ValueError("drop_rate must be in (0, 1]")
        if self.step_size < 1:
            raise ValueError("step_size must be >= 1")
        if self.n_basis < 1:
            raise ValueError("n_basis must be >= 1")
        if self.coord_mode not in COORD_MODES:
            raise ValueError(f"coord_mode must be one of {COORD_MODES}")
        if self.optimizer not in ("adam", "sgd"):
            raise ValueError("optimizer must be 'adam' or 'sgd'")
        for name in ("a0_floor", "sigma_floor"):
            if not getattr(self, name) > 0:
                raise ValueError(f"{name} must be > 0")
        if self.p0_floor < 0:
            raise ValueError("p0_floor must be >= 0")
        if self.prune_every < 1 or self.static_iters < 1 or self.dynamic_iters < 1:
            raise ValueError("iteration counts and prune cadence must be >= 1")
        if self.basis not in BASES:
            raise ValueError(f"basis must be one of {BASES}")


@dataclass
class AdamState:
    """First / second moment buffers and step counter for one parameter."""

    m: object
    v: object
    t: int = 0

    @classmethod
    def like(cls, param) -> "AdamState":
        return cls(np.zeros_like(param), np.zeros_like(param))
