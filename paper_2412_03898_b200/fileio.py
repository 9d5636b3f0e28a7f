"""PAT1 tensor and GGB1 cloud containers.

Byte-compatible with pacloud/fileio.py:40-136 (``write_tensor`` /
``read_tensor`` / ``write_cloud`` / ``read_cloud``), little endian:

  PAT1: b"PAT1", version u32 = 1, dtype u32 = 1 (f32), rank u32,
        dims u64[rank], row-major f32 payload.
  GGB1: b"GGB1", version u32 = 1, ball count u64, basis count N u32,
        descriptor length u32 + b"a0,p0,mu_x,mu_y,mu_z", then per ball
        f32[5 + 7N] = (p0, a0, mu[3], theta[N], sigma[N], omega[5][N]).

Readers validate magic, version, dtype, descriptor and payload length and
return float64; f32 storage makes write -> read -> write byte-stable.  The
headers are packed with numpy structured dtypes (one buffer, no per-field
writes); payloads may come straight from device tensors.
"""

from __future__ import annotations

import numpy as np

from .core import N_CHANNELS, DynamicCloud

TENSOR_MAGIC = b"PAT1"
CLOUD_MAGIC = b"GGB1"
FORMAT_VERSION = 1
DTYPE_F32 = 1
CHANNEL_DESCRIPTOR = "a0,p0,mu_x,mu_y,mu_z"

_TENSOR_HEAD = np.dtype([("magic", "S4"), ("version", "<u4"),
                         ("dtype", "<u4"), ("rank", "<u4")])
_CLOUD_HEAD = np.dtype([("magic", "S4"), ("version", "<u4"),
                        ("n_balls", "<u8"), ("n_basis", "<u4"),
                        ("desc_len", "<u4")])


def _host_f32(a) -> np.ndarray:
    if hasattr(a, "detach"):                       # torch tensor (any device)
        a = a.detach().to("cpu").numpy()
    return np.ascontiguousarray(a, dtype="<f4")


def write_tensor(path, array) -> None:
    """Store an array (numpy or torch) as an f32 PAT1 file."""
    a = _host_f32(array)
    head = np.zeros((), _TENSOR_HEAD)
    head["magic"], head["version"] = TENSOR_MAGIC, FORMAT_VERSION
    head["dtype"], head["rank"] = DTYPE_F32, a.ndim
    with open(path, "wb") as f:
        f.write(head.tobytes())
        f.write(np.asarray(a.shape, dtype="<u8").tobytes())
        f.write(a.tobytes())


def read_tensor(path) -> np.ndarray:
    """Read a PAT1 file into a float64 array."""
    raw = memoryview(open(path, "rb").read())
    if len(raw) < _TENSOR_HEAD.itemsize or bytes(raw[:4]) != TENSOR_MAGIC:
        raise ValueError(f"{path}: not a tensor file (bad magic)")
    head = np.frombuffer(raw, _TENSOR_HEAD, count=1)[0]
    if head["version"] != FORMAT_VERSION:
        raise ValueError(f"{path}: unsupported format version "
                         f"{int(head['version'])}")
    if head["dtype"] != DTYPE_F32:
        raise ValueError(f"{path}: unsupported dtype code "
                         f"{int(head['dtype'])}")
    rank = int(head["rank"])
    start = _TENSOR_HEAD.itemsize + 8 * rank
    dims = tuple(int(d) for d in np.frombuffer(raw, "<u8", count=rank,
                                               offset=_TENSOR_HEAD.itemsize))
    count = int(np.prod(dims)) if rank else 1
    if len(raw) != start + 4 * count:
        raise ValueError(f"{path}: payload length {len(raw) - start} != "
                         f"4 * prod(dims) = {4 * count}")
    return np.frombuffer(raw, "<f4", count=count, offset=start) \
        .astype(np.float64).reshape(dims)


def _as_dynamic(cloud) -> DynamicCloud:
    if hasattr(cloud, "omega"):
        return cloud
    balls = list(cloud)                                # list of GaussBall
    b = len(balls)
    return DynamicCloud(np.array([x.p0 for x in balls], float).reshape(b),
                        np.array([x.a0 for x in balls], float).reshape(b),
                        np.array([x.mu for x in balls], float).reshape(b, 3),
                        np.zeros((b, 0)), np.zeros((b, 0)),
                        np.zeros((b, N_CHANNELS, 0)))


def write_cloud(path, cloud) -> None:
    """Store a DynamicCloud (or a list of GaussBall, basis count 0) as
    GGB1.  Per-channel basis fields have no file representation."""
    c = _as_dynamic(cloud)
    if getattr(c, "basis", "gauss") != "gauss":
        raise ValueError("GGB1 stores Gaussian-basis clouds only; the "
                         "poly+Fourier basis has no file representation")
    theta = np.asarray(c.theta)
    if theta.ndim == 3:
        raise ValueError("per-channel basis fields cannot be serialized; "
                         "share theta and sigma across channels")
    b = len(np.asarray(c.p0))
    nb = np.asarray(c.omega).shape[-1]
    rec = np.empty((b, 5 + (2 + N_CHANNELS) * nb), dtype="<f4")
    rec[:, 0] = np.asarray(c.p0)
    rec[:, 1] = np.asarray(c.a0)
    rec[:, 2:5] = np.asarray(c.mu)
    rec[:, 5:5 + nb] = theta
    rec[:, 5 + nb:5 + 2 * nb] = np.asarray(c.sigma)
    rec[:, 5 + 2 * nb:] = np.asarray(c.omega).reshape(b, N_CHANNELS * nb)
    desc = CHANNEL_DESCRIPTOR.encode()
    head = np.zeros((), _CLOUD_HEAD)
    head["magic"], head["version"] = CLOUD_MAGIC, FORMAT_VERSION
    head["n_balls"], head["n_basis"], head["desc_len"] = b, nb, len(desc)
    with open(path, "wb") as f:
        f.write(head.tobytes())
        f.write(desc)
        f.write(rec.tobytes())


def read_cloud(path) -> DynamicCloud:
    """Read a GGB1 file into a float64 DynamicCloud (shared basis)."""
    raw = memoryview(open(path, "rb").read())
    if len(raw) < _CLOUD_HEAD.itemsize or bytes(raw[:4]) != CLOUD_MAGIC:
        raise ValueError(f"{path}: not a cloud file (bad magic)")
    head = np.frombuffer(raw, _CLOUD_HEAD, count=1)[0]
    if head["version"] != FORMAT_VERSION:
        raise ValueError(f"{path}: unsupported format version "
                         f"{int(head['version'])}")
    b, nb, dl = int(head["n_balls"]), int(head["n_basis"]), int(head["desc_len"])
    start = _CLOUD_HEAD.itemsize + dl
    desc = bytes(raw[_CLOUD_HEAD.itemsize:start]).decode()
    if desc != CHANNEL_DESCRIPTOR:
        raise ValueError(f"{path}: unexpected channel order '{desc}'")
    width = 5 + (2 + N_CHANNELS) * nb
    if len(raw) != start + 4 * width * b:
        raise ValueError(f"{path}: truncated cloud file")
    flat = np.frombuffer(raw, "<f4", count=width * b, offset=start) \
        .astype(np.float64).reshape(b, width)
    return DynamicCloud(flat[:, 0], flat[:, 1], flat[:, 2:5],
                        flat[:, 5:5 + nb], flat[:, 5 + nb:5 + 2 * nb],
                        flat[:, 5 + 2 * nb:].reshape(b, N_CHANNELS, nb))
