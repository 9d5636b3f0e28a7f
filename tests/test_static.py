"""the static stage (reconstruction.py:160-231) against
the live reference's golden run and the oracle restatement."""

import numpy as np
import pytest

import oracle
from helpers import SIGNAL_TOL, rel_l2, small_array
from paper_2412_03898_b200.core import Box, ReconConfig, SensorArray


def _cfg(**kw):
    base = dict(lr_coords=2e-2, lr_pressure=5e-2, lr_std=1e-2,
                static_iters=6, prune_every=3, prune_threshold=0.9,
                init_pitch=1.5, init_p0_scale=0.5, step_size=4, drop_rate=0.5,
                seed=1)
    base.update(kw)
    return ReconConfig(**base)


def test_oracle_static_golden(golden):
    arr = small_array(golden, SensorArray)
    losses = []
    p0, a0, mu = oracle.static_reconstruct(
        golden["static_obs"], arr, _cfg(), -2.5 * np.ones(3),
        2.5 * np.ones(3), losses=losses)
    assert np.allclose(losses, golden["static_loss"], rtol=1e-10)
    assert np.allclose(p0, golden["static_p0"], rtol=1e-9)
    assert np.allclose(a0, golden["static_a0"], rtol=1e-9)
    assert np.allclose(mu, golden["static_mu"], rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_static_reconstruct_golden(pc, golden):
    from paper_2412_03898_b200.static import static_reconstruct
    arr = small_array(golden, SensorArray)
    log = []
    balls = static_reconstruct(golden["static_obs"], arr, _cfg(),
                               Box.cube(2.5), progress=log.append)
    assert [r["n_balls"] for r in log] == list(golden["static_nballs"])
    assert [r["stage"] for r in log] == ["static"] * 6
    assert np.allclose([r["loss"] for r in log], golden["static_loss"],
                       rtol=SIGNAL_TOL)
    p0 = np.array([b.p0 for b in balls])
    a0 = np.array([b.a0 for b in balls])
    mu = np.array([b.mu for b in balls])
    assert len(balls) == len(golden["static_p0"])
    assert rel_l2(p0, golden["static_p0"]) < 1e-5
    assert rel_l2(a0, golden["static_a0"]) < 1e-5
    assert rel_l2(mu, golden["static_mu"]) < 1e-5


@pytest.mark.gpu
def test_static_reconstruct_vs_oracle_planar(pc):
    """A larger static fit (planar grid, config-1 geometry at reduced size)
    with pruning, SGD and Adam."""
    from paper_2412_03898_b200 import synth
    from paper_2412_03898_b200.static import static_reconstruct
    prob = synth.make_problem(1, n_balls=60, n_sensors=64, n_samples=1024)
    arr = prob.array
    a0, p0, mu = prob.gt_frames[0]
    obs = oracle.forward_frame(oracle.States(a0, p0, mu), arr)
    obs = obs.astype(np.float32).astype(np.float64)
    lo, hi = mu.min(0) - 1.0, mu.max(0) + 1.0
    for opt in ("adam", "sgd"):
        cfg = ReconConfig(lr_coords=1e-3, lr_pressure=1e-2, lr_std=1e-3,
                          static_iters=8, prune_every=4, prune_threshold=0.3,
                          init_pitch=3.0, init_p0_scale=0.2, optimizer=opt)
        losses = []
        want = oracle.static_reconstruct(obs, arr, cfg, lo, hi, losses=losses)
        log = []
        balls = static_reconstruct(obs, arr, cfg, Box(lo, hi),
                                   progress=log.append)
        got_l = np.array([r["loss"] for r in log])
        assert np.abs(got_l - losses).max() < SIGNAL_TOL * max(losses), opt
        assert len(balls) == len(want[0]), opt
        got = np.array([[b.p0, b.a0, *b.mu] for b in balls])
        ref = np.column_stack([want[0], want[1], want[2]])
        assert rel_l2(got, ref) < 1e-5, opt


@pytest.mark.gpu
def test_static_errors(pc, golden):
    from paper_2412_03898_b200.static import StaticEngine, static_reconstruct
    arr = small_array(golden, SensorArray)
    with pytest.raises(ValueError):
        static_reconstruct(np.zeros((3, 3)), arr, _cfg(), Box.cube(2.5))
    # every ball pruned -> RuntimeError (zero data: p0 = 0, max = 0)
    with pytest.raises(RuntimeError):
        static_reconstruct(np.zeros((arr.n_sensors, arr.n_samples)), arr,
                           _cfg(static_iters=3, prune_every=1), Box.cube(2.5))
    # non-finite gradient names the group; earlier groups already stepped
    eng = StaticEngine(np.ones(2), np.ones(2), np.zeros((2, 3)) + 1.0, arr,
                       np.zeros((arr.n_sensors, arr.n_samples)), _cfg())
    eng._grads()
    import torch
    p_before = eng.P.clone()
    orig = eng._grads

    def poisoned():
        orig()
        eng.Gf[2 * eng.B] = float("nan")
    eng._grads = poisoned
    with pytest.raises(ValueError, match="coords"):
        eng.iterate(0)
    assert not torch.equal(eng.P[:2 * eng.B], p_before[:2 * eng.B])
    assert torch.equal(eng.P[2 * eng.B:], p_before[2 * eng.B:])
