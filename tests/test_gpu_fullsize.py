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


def _subarray(arr, every):
    from paper_2412_03898_b200.core import SensorArray
    return SensorArray(arr.positions[::every], arr.sound_speed,
                       arr.sample_rate, arr.n_samples, arr.t_start)


def test_config3_full_iteration_vs_oracle(pc):
    """One full BASELINE config-3 engine iteration — all 200,000 balls, all
    32 frames, poly+Fourier deformation, forward + loss + adjoint + fused
    deformation backward — against the oracle's frame loop
    (reconstruction.py:293-316) on a 16-sensor subsample of the 1,024."""
    from paper_2412_03898_b200 import synth
    from paper_2412_03898_b200.engine import IterationEngine
    from paper_2412_03898_b200.radiator import DeviceArray, forward_device
    prob = synth.make_problem(3)
    sub = _subarray(prob.array, 64)
    darr = DeviceArray(sub, 6.0, False)
    obs = []
    for a, p, m in prob.gt_frames:          # observed traces (input only)
        mm, aa, pp = _dev(m, a, p)
        obs.append(forward_device(darr, mm, aa, pp)[0][0].cpu().numpy())
    obs = np.stack(obs).astype(np.float32)
    frames = np.arange(prob.n_frames)
    eng = IterationEngine(prob.cloud, sub, obs, prob.frame_times, prob.config)
    eng.compute_grads(frames)
    loss, flags, _ = eng.check_and_status()
    g = eng.grads_numpy()
    ref_loss, ref = oracle.iteration_grads(
        prob.cloud, prob.frame_times, obs.astype(np.float64), sub,
        prob.config, basis=prob.cloud.basis)
    assert not flags.any()
    assert abs(loss - ref_loss) / ref_loss < SIGNAL_TOL
    for k in ("p0", "a0", "mu", "omega"):
        assert rel_l2(g[k], getattr(ref, k)) < GRAD_TOL, k


def test_config4_forward_256_sensors_adjoint_64(pc):
    """BASELINE config 4 (1,000,000 balls, 60 mm hemisphere, T = 8192):
    forward on 256 of the 2,048 sensors and adjoint on 64, full cloud."""
    arr, sub, a0, p0, mu = _frame(4, 8)
    st = oracle.States(a0, p0, mu)
    ref = oracle.forward_frame(st, sub)
    got = pc.forward_frame(pc.CloudState(a0, p0, mu), sub)
    assert rel_l2(got, ref) < SIGNAL_TOL
    sub64 = _subarray(arr, 32)
    rng = np.random.default_rng(44)
    res = rng.normal(0, 1e-2, (64, arr.n_samples))
    res = res.astype(np.float32).astype(np.float64)
    g_ref = oracle.frame_state_grads(st, sub64, res)
    g = pc.frame_state_grads(pc.CloudState(a0, p0, mu), sub64, res)
    for c in range(5):
        assert rel_l2(g[:, c], g_ref[:, c]) < GRAD_TOL, c
