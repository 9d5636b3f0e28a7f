"""The reference's end-to-end finite-difference problem
(test_radiator.py:187-226) restated on the oracle: 3 balls, 8 sensors,
64 samples, Gaussian basis N=3, one frame at t=0.55."""

import numpy as np

import oracle
from paper_2412_03898_b200.synth import fibonacci_sphere


def end_to_end_problem(pc, rng, mode):
    arr = pc.SensorArray(fibonacci_sphere(8, 30.0), 1.5, 6.0, 64, 16.0)
    n_balls, nb = 3, 3
    observed = rng.normal(0, 1e-4, (8, 64))
    p0 = rng.uniform(0.4, 1.2, n_balls)
    a0 = rng.uniform(0.4, 1.0, n_balls)
    mu = rng.uniform(-4, 4, (n_balls, 3))
    theta = np.tile(np.linspace(0, 1, nb), (n_balls, 1))
    sigma = np.full((n_balls, nb), 0.4)
    omega = rng.uniform(-0.2, 0.2, (n_balls, 5, nb))
    x0 = np.concatenate([p0, a0, mu.ravel(), theta.ravel(), sigma.ravel(),
                         omega.ravel()])

    def unpack(x):
        i = 0
        _p0 = x[i:i + n_balls]; i += n_balls
        _a0 = x[i:i + n_balls]; i += n_balls
        _mu = x[i:i + 3 * n_balls].reshape(n_balls, 3); i += 3 * n_balls
        _th = x[i:i + n_balls * nb].reshape(n_balls, nb); i += n_balls * nb
        _sg = x[i:i + n_balls * nb].reshape(n_balls, nb); i += n_balls * nb
        return pc.DynamicCloud(_p0, _a0, _mu, _th, _sg,
                               x[i:].reshape(n_balls, 5, nb))

    def total_loss(x):
        st = oracle.cloud_states_at(unpack(x), 0.55, mode)
        pred = oracle.forward_frame(st, arr, exact=True)
        return 0.5 * float(np.sum((pred - observed) ** 2))

    return arr, observed, x0, unpack, total_loss
