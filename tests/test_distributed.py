"""Multi-rank host logic on CPU: world_size 2 over gloo.

The exchange (distributed.allreduce_iteration) and the shard maps
(shard_range / frame_shard) are the code the NCCL path runs; here the
per-rank compute is the CPU oracle, so the test checks that frame- and
sensor-sharded gradients reduce to the single-process result and that the
replicated Adam step keeps the ranks bit-identical.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2412_03898_b200.core import SensorArray
from paper_2412_03898_b200.distributed import (allreduce_iteration,
                                               frame_shard, shard_range)
from paper_2412_03898_b200.synth import make_problem


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for n in (0, 1, 7, 8, 32, 2048):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(n, r, world)
                seen += list(range(lo, hi))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_frame_shard_of_selected_minibatch():
    sel = np.array([1, 4, 5, 9, 11])
    got = np.concatenate([frame_shard(sel, r, 2) for r in range(2)])
    assert np.array_equal(got, sel)


def _problem():
    prob = make_problem(3, seed=11, n_balls=120, n_sensors=24, n_frames=4,
                        n_samples=4096)
    obs = np.stack([oracle.forward_frame(oracle.States(a, p, m), prob.array)
                    for a, p, m in prob.gt_frames])
    return prob, obs.astype(np.float32).astype(np.float64)


def _flat(g):
    return np.concatenate([g.p0.ravel(), g.a0.ravel(), g.mu.ravel(),
                           g.omega.ravel()])


def _worker(rank, world, port, mode, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob, obs = _problem()
        cfg = prob.config
        frames = np.arange(prob.n_frames)
        arr = prob.array
        if mode == "frames":
            mine = frame_shard(frames, rank, world)
            loss, g = oracle.iteration_grads(
                prob.cloud, prob.frame_times[mine], obs[mine], arr, cfg,
                basis=prob.cloud.basis, threads=1)
        else:
            lo, hi = shard_range(arr.n_sensors, rank, world)
            sub = SensorArray(arr.positions[lo:hi], arr.sound_speed,
                              arr.sample_rate, arr.n_samples, arr.t_start)
            loss, g = oracle.iteration_grads(
                prob.cloud, prob.frame_times, obs[:, lo:hi], sub, cfg,
                basis=prob.cloud.basis, threads=1)
        grads = torch.as_tensor(_flat(g))
        loss_t = torch.tensor([loss], dtype=torch.float64)
        coinc = torch.tensor([(1 << 63) - 1 - rank], dtype=torch.int64)
        allreduce_iteration(grads, loss_t, coinc)
        # replicated Adam on every rank
        p = torch.as_tensor(np.concatenate([prob.cloud.p0, prob.cloud.a0,
                                            prob.cloud.mu.ravel(),
                                            prob.cloud.omega.ravel()]))
        pn = p.numpy().copy()
        st = oracle.Moments(np.zeros_like(pn), np.zeros_like(pn))
        oracle.adam_step(pn, grads.numpy(), st, 1e-3)
        gathered = [torch.zeros_like(p) for _ in range(world)]
        dist.all_gather(gathered, torch.as_tensor(pn))
        if rank == 0:
            np.savez(out_path, grads=grads.numpy(), loss=loss_t.numpy(),
                     coinc=coinc.numpy(),
                     params=np.stack([x.numpy() for x in gathered]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["frames", "sensors"])
def test_sharded_gradients_match_single_process(tmp_path, mode):
    out = tmp_path / f"{mode}.npz"
    mp.spawn(_worker, args=(2, _free_port(), mode, str(out)), nprocs=2,
             join=True)
    res = np.load(out)
    prob, obs = _problem()
    loss, g = oracle.iteration_grads(prob.cloud, prob.frame_times, obs,
                                     prob.array, prob.config,
                                     basis=prob.cloud.basis, threads=1)
    full = _flat(g)
    assert abs(res["loss"][0] - loss) <= 1e-12 * abs(loss)
    assert np.linalg.norm(res["grads"] - full) <= 1e-12 * np.linalg.norm(full)
    assert int(res["coinc"][0]) == (1 << 63) - 2          # MIN over ranks
    assert np.array_equal(res["params"][0], res["params"][1])


def test_ball_orders_are_permutations_and_hilbert_has_unit_steps():
    """engine.hilbert_order (the internal ball layout): a permutation; on a
    full 2^b lattice consecutive cells are face neighbours (the property the
    32-ball culling groups rely on), which the Z-order lacks."""
    from paper_2412_03898_b200.engine import hilbert_order, morton_order
    g = np.stack(np.meshgrid(np.arange(16), np.arange(16), np.arange(16),
                             indexing="ij"), -1).reshape(-1, 3).astype(float)
    for fn in (hilbert_order, morton_order):
        o = fn(g, bits=4)
        assert sorted(o.tolist()) == list(range(len(g)))
    steps = np.abs(np.diff(g[hilbert_order(g, bits=4)], axis=0)).sum(axis=1)
    assert (steps == 1).all()
    rng = np.random.default_rng(3)
    mu = rng.uniform(-20, 20, (5000, 3))
    o = hilbert_order(mu)
    assert sorted(o.tolist()) == list(range(5000))
    ext = lambda order: np.mean(np.ptp(mu[order][:4992].reshape(-1, 32, 3), axis=1).max(axis=1))
    assert ext(o) <= ext(morton_order(mu))
    assert len(hilbert_order(np.zeros((0, 3)))) == 0
    # the engine's layout: Hilbert runs of 64 balls, radius-sorted inside
    from paper_2412_03898_b200.engine import spatial_ball_order
    a0 = rng.uniform(0.1, 0.5, 5000)
    s = spatial_ball_order(mu, a0)
    assert sorted(s.tolist()) == list(range(5000))
    for k in range(0, 5000, 64):
        assert set(s[k:k + 64]) == set(o[k:k + 64])
        assert (np.diff(a0[s[k:k + 64]]) >= 0).all()
    assert len(spatial_ball_order(np.zeros((0, 3)), np.zeros(0))) == 0
