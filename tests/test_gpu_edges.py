"""Kernel-path edge cases against the oracle: arrival ranges longer than one
shared-memory segment (balls straddling segment boundaries), odd T (the
unaligned adjoint and scalar epilogue), sensor counts that are not multiples
of the warp / CTA tiling, batched frames, and the T >= 32768 rejection."""

import numpy as np
import pytest

import oracle
from helpers import GRAD_TOL, SIGNAL_TOL, rel_l2

pytestmark = pytest.mark.gpu


def _cloud(rng, B, half, a_lo, a_hi):
    return (rng.uniform(a_lo, a_hi, B), rng.uniform(0.2, 1.0, B),
            rng.uniform(-half, half, (B, 3)))


def _check_frame(pc, a0, p0, mu, arr, rng):
    st = pc.CloudState(a0, p0, mu)
    ref = oracle.forward_frame(oracle.States(a0, p0, mu), arr)
    got = pc.forward_frame(st, arr)
    assert rel_l2(got, ref) < SIGNAL_TOL
    res = rng.normal(0, 1e-2, ref.shape).astype(np.float32).astype(np.float64)
    g_ref = oracle.frame_state_grads(oracle.States(a0, p0, mu), arr, res)
    g = pc.frame_state_grads(st, arr, res)
    for c in range(5):
        assert rel_l2(g[:, c], g_ref[:, c]) < GRAD_TOL, c


def test_arrival_range_spans_several_segments(pc):
    """60 mm hemisphere around a +-30 mm cube at 40 MHz: the arrival range
    per sensor (~2800 samples) exceeds the 1536-sample segment cap."""
    from paper_2412_03898_b200.geometry import fibonacci_sphere
    rng = np.random.default_rng(12)
    pos = fibonacci_sphere(64, 60.0)[:40]
    arr = pc.SensorArray(pos, 1.5, 40.0, 8192, 0.0)
    a0, p0, mu = _cloud(rng, 400, 30.0, 0.2, 0.6)
    _check_frame(pc, a0, p0, mu, arr, rng)


def test_odd_samples_and_ragged_sensor_count(pc):
    from paper_2412_03898_b200.geometry import fibonacci_sphere
    rng = np.random.default_rng(13)
    pos = fibonacci_sphere(74, 25.0)[:37]           # 37 sensors
    arr = pc.SensorArray(pos, 1.5, 20.0, 1001, 8.0)  # odd T
    a0, p0, mu = _cloud(rng, 157, 6.0, 0.25, 0.7)
    _check_frame(pc, a0, p0, mu, arr, rng)


def test_batched_frames_match_per_frame(pc):
    """pc_forward_traces / pc_residual_state_grads over F frames at once
    equal F single-frame calls (frame index only selects states)."""
    import torch
    from paper_2412_03898_b200.radiator import (DeviceArray, forward_device,
                                                state_grads_device)
    from paper_2412_03898_b200.geometry import fibonacci_sphere
    rng = np.random.default_rng(14)
    arr = pc.SensorArray(fibonacci_sphere(96, 30.0)[:48], 1.5, 30.0, 2048, 6.0)
    darr = DeviceArray(arr, 6.0, False)
    F, B = 3, 230
    mu = torch.as_tensor(rng.uniform(-5, 5, (F, B, 3)), device="cuda")
    a0 = torch.as_tensor(rng.uniform(0.2, 0.6, (F, B)), dtype=torch.float32,
                         device="cuda")
    p0 = torch.as_tensor(rng.uniform(0.2, 1.0, (F, B)), dtype=torch.float32,
                         device="cuda")
    out, _, _ = forward_device(darr, mu, a0, p0)
    G, _ = state_grads_device(darr, mu, a0, p0, out)[:2]
    for f in range(F):
        o1, _, _ = forward_device(darr, mu[f:f + 1].contiguous(),
                                  a0[f:f + 1].contiguous(),
                                  p0[f:f + 1].contiguous())
        assert torch.equal(o1[0], out[f])
        g1 = state_grads_device(darr, mu[f:f + 1].contiguous(),
                                a0[f:f + 1].contiguous(),
                                p0[f:f + 1].contiguous(), o1)[0]
        assert torch.equal(g1[0], G[f])


def test_long_traces(pc):
    """T beyond 2^15 samples (window indices are segment-relative in the
    forward and full-width in the adjoint)."""
    rng = np.random.default_rng(15)
    pos = np.array([[0.0, 0.0, 300.0], [5.0, 0.0, 400.0], [0.0, 5.0, 600.0]])
    arr = pc.SensorArray(pos, 1.5, 40.0, 40001, 0.0)      # 40001 samples, odd
    a0, p0, mu = _cloud(rng, 60, 4.0, 0.2, 0.6)
    _check_frame(pc, a0, p0, mu, arr, rng)
