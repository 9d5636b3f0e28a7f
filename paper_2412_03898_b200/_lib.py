"""ctypes binding of libpacloud_b200.so (the C ABI in include/pacloud_b200.h).

Device memory and streams come from PyTorch (plumbing only); every compute
call goes through this library.  There is no CPU fallback: a missing library
or a missing CUDA device raises at first use.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_int32, c_int64,
                    c_size_t, c_void_p)
from pathlib import Path

import torch

LIB_NAME = "libpacloud_b200.so"
LIB_PATH = Path(__file__).resolve().with_name(LIB_NAME)

PC_OK = 0
PC_COORD = {"multiplicative": 0, "additive": 1, "radial": 2}
PC_BASIS = {"gauss": 0, "polyfourier": 1}
PC_MAX_SEGMENTS = 16
INT64_MAX = (1 << 63) - 1


class PcArray(Structure):
    _fields_ = [("positions", c_void_p), ("n_sensors", c_int32),
                ("n_samples", c_int32), ("sound_speed", c_double),
                ("t_start", c_double), ("dt", c_double),
                ("support_sigmas", c_double), ("exact", c_int32),
                ("sensor_offset", c_int32), ("sensor_order", c_void_p),
                ("n_sensors_total", c_int32), ("frame_offset", c_int32)]


class PcCloud(Structure):
    _fields_ = [("p0", c_void_p), ("a0", c_void_p), ("mu", c_void_p),
                ("theta", c_void_p), ("sigma", c_void_p),
                ("omega", c_void_p), ("n_balls", c_int64),
                ("n_basis", c_int32), ("per_channel", c_int32),
                ("basis_kind", c_int32), ("reserved", c_int32)]


class PcCloudGrads(Structure):
    _fields_ = [("p0", c_void_p), ("a0", c_void_p), ("mu", c_void_p),
                ("theta", c_void_p), ("sigma", c_void_p),
                ("omega", c_void_p)]


# (name, restype, argtypes) for every symbol include/pacloud_b200.h declares
_P = c_void_p
SIGNATURES = {
    "pc_deform_states": (c_int32, [POINTER(PcCloud), _P, c_int32, c_int32,
                                   c_double, _P, _P, _P, _P, _P]),
    "pc_deform_states_f64": (c_int32, [POINTER(PcCloud), _P, c_int32,
                                       c_int32, c_double, _P, _P, _P, _P]),
    "pc_eval_basis": (c_int32, [_P, _P, _P, c_int64, _P, _P]),
    "pc_eval_h": (c_int32, [c_double, _P, _P, _P, c_int32, _P, _P]),
    "pc_deform_jacobian": (c_int32, [POINTER(PcCloud), c_double, c_int32,
                                     c_double, _P, _P, _P, _P, _P]),
    "pc_assemble_grads": (c_int32, [_P, c_int64, c_int32, _P, _P, _P, _P,
                                    POINTER(c_int32), c_int32, c_int32, _P,
                                    _P, _P, _P, _P, _P, _P]),
    "pc_deform_backward": (c_int32, [POINTER(PcCloud), _P, c_int32, c_int32,
                                     c_double, _P, _P, POINTER(PcCloudGrads),
                                     _P]),
    "pc_forward_plan": (c_int32, [c_int64, c_int32, POINTER(PcArray),
                                  POINTER(c_int32)]),
    "pc_forward_variant": (c_int32, [POINTER(PcArray)]),
    "pc_forward_workspace_bytes": (c_size_t, [c_int64, c_int32,
                                              POINTER(PcArray)]),
    "pc_forward_traces": (c_int32, [_P, _P, _P, c_int64, c_int32,
                                    POINTER(PcArray), _P, _P, _P, _P, _P,
                                    c_size_t, _P]),
    "pc_residual_state_grads": (c_int32, [_P, _P, _P, c_int64, c_int32,
                                          POINTER(PcArray), _P, _P, _P, _P]),
    "pc_residual_loss": (c_int32, [_P, _P, _P, _P, _P, c_int32, c_int32,
                                   c_int32, _P]),
    "pc_pressure_kernel": (c_int32, [_P, _P, _P, _P, c_int64, c_double, _P,
                                     _P, _P, _P, _P]),
    "pc_voxelize_workspace_bytes": (c_size_t, [c_int64]),
    "pc_voxelize": (c_int32, [_P, _P, _P, c_int64, POINTER(c_double),
                              c_double, POINTER(c_int32), c_double, c_int32,
                              _P, _P, _P, c_size_t, _P]),
    "pc_ubp_filter": (c_int32, [_P, c_int32, c_int32, c_double, c_double, _P,
                                _P]),
    "pc_backproject": (c_int32, [_P, _P, c_int32, c_int32, c_double, c_double,
                                 c_double, POINTER(c_double), c_double,
                                 POINTER(c_int32), _P, _P]),
    "pc_update_guarded": (c_int32, [_P, _P, _P, _P, c_int32, POINTER(c_int64),
                                    POINTER(c_double), POINTER(c_int32), _P,
                                    _P, _P, _P, c_int32, _P]),
    "pc_l2_loss": (c_int32, [_P, _P, c_int64, _P, _P]),
    "pc_check_finite": (c_int32, [_P, c_int32, POINTER(c_int64), _P, _P]),
    "pc_adam_segments": (c_int32, [_P, _P, _P, _P, c_int32, POINTER(c_int64),
                                   POINTER(c_double), POINTER(c_int32),
                                   POINTER(c_double), _P]),
    "pc_sgd_segments": (c_int32, [_P, _P, c_int32, POINTER(c_int64),
                                  POINTER(c_double), POINTER(c_double), _P]),
    "pc_check_finite_f64": (c_int32, [_P, c_int32, POINTER(c_int64), _P,
                                      _P]),
    "pc_adam_segments_f64": (c_int32, [_P, _P, _P, _P, c_int32,
                                       POINTER(c_int64), POINTER(c_double),
                                       POINTER(c_int32), POINTER(c_double),
                                       _P]),
    "pc_sgd_segments_f64": (c_int32, [_P, _P, c_int32, POINTER(c_int64),
                                      POINTER(c_double), POINTER(c_double),
                                      _P]),
    "pc_compact_workspace_bytes": (c_size_t, [c_int64]),
    "pc_prune_mask": (c_int32, [_P, c_int64, c_double, _P, _P, _P, c_size_t,
                                _P]),
    "pc_compact_index": (c_int32, [_P, _P, c_int64, _P, _P, _P, c_size_t,
                                   _P]),
    "pc_densify_masks": (c_int32, [_P, _P, c_int64, c_double, _P, _P,
                                   _P, _P, _P]),
    "pc_abs_quantile_workspace_bytes": (c_size_t, []),
    "pc_abs_quantile_f32": (c_int32, [_P, c_int64, c_int64, c_double, _P, _P,
                                      c_size_t, _P]),
    "pc_densify_flags": (c_int32, [_P, c_int64, c_int64, c_int64, _P, _P, _P,
                                   _P]),
    "pc_densify_apply": (c_int32, [_P, _P, _P, _P, _P, c_int64, c_double,
                                   _P]),
    "pc_gather_rows": (c_int32, [_P, _P, _P, c_int64, c_int64, _P]),
    "pc_version": (c_char_p, []),
}

_lib = None


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing or no CUDA device is available."""


def load_library(require_cuda: bool = True):
    """Load libpacloud_b200.so (and check for a CUDA device)."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("PACLOUD_B200_LIB", LIB_PATH))
        if not path.exists():
            raise NativeLibraryError(
                f"{path} is not built; run `python -c 'import __graft_entry__ "
                f"as g; g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise NativeLibraryError(
            "paper_2412_03898_b200 needs a CUDA device (sm_100a); there is no "
            "CPU fallback")
    return _lib


def check(status: int, what: str) -> None:
    if status != PC_OK:
        raise RuntimeError(f"{what} failed (pacloud_b200 status {status})")


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None / empty)."""
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def i64_array(vals):
    return (c_int64 * len(vals))(*[int(v) for v in vals])


def f64_array(vals):
    return (c_double * len(vals))(*[float(v) for v in vals])


def i32_array(vals):
    return (c_int32 * len(vals))(*[int(v) for v in vals])
