"""Full-size BASELINE workloads (configs 2-4, one frame) through the C ABI:
oracle parity on a sensor subsample (every ball, exact inputs), and the
size-independent properties the physics gives — p0 scaling and residual
scaling are exact (every term scales by a power of two), superposition of two
clouds holds to fp32 rounding."""

import numpy as np
import pytest
import torch

import oracle
from helpers import GRAD_TOL, SIGNAL_TOL, rel_l2

pytestmark = pytest.mark.gpu


def _frame(cfg, every):
    from paper_2412_03898_b200 import synth
    from paper_2412_03898_b200.core import SensorArray
    prob = synth.make_problem(cfg, seed=cfg)
    arr = prob.array
    sub = SensorArray(arr.positions[::every], arr.sound_speed, arr.sample_rate,
                      arr.n_samples, arr.t_start)
    a0, p0, mu = prob.gt_frames[0]
    q = lambda x: np.asarray(x, np.float32).astype(np.float64)  # noqa: E731
    return arr, sub, q(a0), q(p0), mu


def _dev(mu, a0, p0):
    return (torch.as_tensor(mu, device="cuda")[None].contiguous(),
            torch.as_tensor(a0, dtype=torch.float32, device="cuda")[None].contiguous(),
            torch.as_tensor(p0, dtype=torch.float32, device="cuda")[None].contiguous())


@pytest.mark.parametrize("cfg,every", [(2, 16), (3, 64), (4, 128)])
def test_full_cloud_vs_oracle_on_sensor_subsample(pc, cfg, every):
    arr, sub, a0, p0, mu = _frame(cfg, every)
    st = oracle.States(a0, p0, mu)
    ref = oracle.forward_frame(st, sub)
    got = pc.forward_frame(pc.CloudState(a0, p0, mu), sub)
    assert rel_l2(got, ref) < SIGNAL_TOL
    rng = np.random.default_rng(cfg)
    res = rng.normal(0, 1e-2, ref.shape).astype(np.float32).astype(np.float64)
    g_ref = oracle.frame_state_grads(st, sub, res)
    g = pc.frame_state_grads(pc.CloudState(a0, p0, mu), sub, res)
    for c in range(5):
        assert rel_l2(g[:, c], g_ref[:, c]) < GRAD_TOL, c


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_exact_scalings_and_superposition(pc, cfg):
    from paper_2412_03898_b200.radiator import (DeviceArray, forward_device,
                                                state_grads_device)
    arr, _, a0, p0, mu = _frame(cfg, 1)
    darr = DeviceArray(arr, 6.0, False)
    m, a, p = _dev(mu, a0, p0)
    out, _, _ = forward_device(darr, m, a, p)
    out2, _, _ = forward_device(darr, m, a, p * 2)
    assert torch.equal(out2, out * 2)                  # p0 scaling: exact
    G, _ = state_grads_device(darr, m, a, p, out)
    G2, _ = state_grads_device(darr, m, a, p, out * 2)
    assert torch.equal(G2, G * 2)                      # residual scaling: exact
    # superposition: the cloud split in two halves
    half = len(a0) // 2
    parts = []
    for sl in (slice(0, half), slice(half, None)):
        mm, aa, pp = _dev(mu[sl], a0[sl], p0[sl])
        parts.append(forward_device(darr, mm, aa, pp)[0])
    both = (parts[0].double() + parts[1].double()).cpu().numpy()
    assert rel_l2(out.double().cpu().numpy(), both) < 1e-6


def test_small_grid_sensor_split_adjoint(pc):
    """Grids under two waves split each ball's sensors over two CTAs whose
    partial G add into zeroed output: oracle parity, and two launches are
    bit-identical (two addends onto 0 commute exactly)."""
    from paper_2412_03898_b200.core import SensorArray
    from paper_2412_03898_b200.radiator import DeviceArray, state_grads_device
    arr, _, a0, p0, mu = _frame(1, 1)          # config 1: 256 planar sensors
    keep = slice(0, 600)                       # 150 CTAs: split
    a0, p0, mu = a0[keep], p0[keep], mu[keep]
    st = oracle.States(a0, p0, mu)
    rng = np.random.default_rng(5)
    res = rng.normal(0, 1e-2, (arr.n_sensors, arr.n_samples))
    res = res.astype(np.float32).astype(np.float64)
    g_ref = oracle.frame_state_grads(st, arr, res)
    darr = DeviceArray(arr, 6.0, False)
    m, a, p = _dev(mu, a0, p0)
    r = torch.as_tensor(res, dtype=torch.float32, device="cuda")[None].contiguous()
    G1, _ = state_grads_device(darr, m, a, p, r)
    G2, _ = state_grads_device(darr, m, a, p, r)
    assert torch.equal(G1, G2)
    g = G1[0].double().cpu().numpy()
    for c in range(5):
        assert rel_l2(g[:, c], g_ref[:, c]) < GRAD_TOL, c
