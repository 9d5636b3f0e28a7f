"""The sharded IterationEngine against the single-rank engine (GPU).

Two ranks share the one B200 over gloo (PC_DIST_BACKEND-style functional
check: each rank is its own process with its own CUDA context; the
exchange is distributed.allreduce_iteration).  Frame sharding on reduced
configs 2 and 5, sensor sharding on reduced config 4:

* the loss of every iteration equals the single-rank loss (rel 1e-12),
* the flat parameter gradient of the first iteration matches (rel-L2 1e-6),
* after three Adam steps both ranks hold bit-identical parameters, equal to
  the single-rank parameters (rel-L2 1e-6),
* a coincidence placed in frame 2 (owned by rank 1 / in rank 1's sensor
  block) raises the reference's message (radiator.py:186-192) on BOTH ranks
  for the closest pair of THAT frame, and nothing is updated.

reconstruction.py:303-316 is the loop being sharded.
"""

import dataclasses
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(case):
    from paper_2412_03898_b200 import synth
    if case == "c2":
        prob = synth.make_problem(2, seed=21, n_balls=400, n_sensors=48,
                                  n_frames=4)
    elif case == "c5":
        prob = synth.make_problem(5, seed=22, n_balls=500, n_sensors=40,
                                  n_frames=5)
    else:
        prob = synth.make_problem(4, seed=23, n_balls=600, n_sensors=64,
                                  n_frames=3, n_samples=8192)
    obs = np.stack([oracle.forward_frame(oracle.States(a, p, m), prob.array)
                    for a, p, m in prob.gt_frames]).astype(np.float32)
    return prob, obs


def _coincident_problem():
    """5 frames, additive coordinates; ball 7 reaches sensor m* exactly at
    frame 2 (t = 0.5) through the linear basis term (exact dyadic values)."""
    from paper_2412_03898_b200 import synth
    prob = synth.make_problem(2, seed=24, n_balls=64, n_sensors=16,
                              n_frames=5)
    cl = prob.cloud
    pos = np.asarray(prob.array.positions, dtype=np.float64)
    m_star = 12                                  # in rank 1's sensor block
    cl.omega[:] = 0.0
    cl.mu[7] = pos[m_star]
    cl.mu[7, 0] = pos[m_star, 0] - 0.25
    cl.omega[7, 2, 1] = 0.5                      # x channel, basis t: +0.25 at t=0.5
    cfg = dataclasses.replace(prob.config, coord_mode="additive")
    obs = np.zeros((5, 16, prob.array.n_samples), dtype=np.float32)
    return prob, cfg, obs, m_star


def _run(case, shard, rank, world, iters=3):
    from paper_2412_03898_b200.engine import IterationEngine
    prob, obs = _problem(case)
    eng = IterationEngine(prob.cloud, prob.array, obs, prob.frame_times,
                          prob.config, shard=shard)
    frames = np.arange(prob.n_frames)
    losses, g0 = [], None
    for it in range(iters):
        losses.append(eng.iterate(it, frames))
        if it == 0:
            g0 = eng.Gf.double().cpu().numpy().copy()
    return np.array(losses), g0, eng.P.cpu().numpy().copy()


def _coinc_run(shard, rank, world):
    from paper_2412_03898_b200.engine import IterationEngine
    prob, cfg, obs, _ = _coincident_problem()
    eng = IterationEngine(prob.cloud, prob.array, obs, prob.frame_times,
                          cfg, shard=shard)
    P0 = eng.P.cpu().numpy().copy()
    try:
        eng.iterate(0, np.arange(prob.n_frames))
        msg = ""
    except ValueError as e:
        msg = str(e)
    return msg, bool(np.array_equal(P0, eng.P.cpu().numpy()))


def _worker(rank, world, port, case, shard, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "coinc":
            msg, same = _coinc_run(shard, rank, world)
            np.savez(out.format(rank), msg=np.array(msg), same=same)
        else:
            losses, g0, P = _run(case, shard, rank, world)
            np.savez(out.format(rank), losses=losses, g0=g0, P=P)
    finally:
        torch.distributed.destroy_process_group()


def _spawn(tmp_path, case, shard):
    out = str(tmp_path / (f"{case}_{shard}" + "_r{}.npz"))
    mp.spawn(_worker, args=(2, _free_port(), case, shard, out), nprocs=2,
             join=True)
    return [dict(np.load(out.format(r))) for r in range(2)]


@pytest.mark.parametrize("case,shard", [("c2", "frames"), ("c5", "frames"),
                                        ("c4", "sensors")])
def test_sharded_engine_matches_single_rank(tmp_path, case, shard):
    ranks = _spawn(tmp_path, case, shard)
    losses, g0, P = _run(case, None, 0, 1)
    for r in ranks:
        # iteration 0: same parameters, the loss differs only in the order
        # of the fp64 frame sum; later iterations follow parameters stepped
        # from float32 all-reduced gradients (rounding ~1e-7 of a step)
        assert abs(r["losses"][0] - losses[0]) <= 1e-12 * abs(losses[0]), \
            (r["losses"], losses)
        assert np.allclose(r["losses"], losses, rtol=1e-9, atol=0), \
            (r["losses"] - losses, losses)
        assert np.linalg.norm(r["g0"] - g0) <= 1e-6 * np.linalg.norm(g0)
        assert np.linalg.norm(r["P"] - P) <= 1e-6 * np.linalg.norm(P)
    assert np.array_equal(ranks[0]["P"], ranks[1]["P"])


@pytest.mark.parametrize("shard", ["frames", "sensors"])
def test_sharded_coincidence_names_frame_pair(tmp_path, shard):
    prob, cfg, _, m_star = _coincident_problem()
    # the reference's message: closest pair of frame 2's states
    st = oracle.cloud_states_at(prob.cloud, float(prob.frame_times[2]),
                                "additive", cfg.a0_floor, basis="polyfourier")
    pos = np.asarray(prob.array.positions, dtype=np.float64)
    d = np.linalg.norm(st.mu_t[:, None, :] - pos[None, :, :], axis=2)
    b, m = np.unravel_index(np.argmin(d), d.shape)
    assert (b, m) == (7, m_star)
    ranks = _spawn(tmp_path, "coinc", shard)
    for r in ranks:
        msg = str(r["msg"])
        assert re.match(rf"ball 7 coincides with sensor {m_star} ", msg), msg
        assert bool(r["same"]), "a coincident iteration must update nothing"
