"""Pin the CPU oracle (test infrastructure) to the reference.

* golden vectors produced by the live reference (tests/golden/make_golden.py)
* the reference test suite's known-answer values
* (build container only) direct comparison with the live reference
"""

import math

import numpy as np
import pytest

import oracle
from helpers import planar_array, rel_l2, small_array


class Arr:
    def __init__(self, positions, sound_speed, sample_rate, n_samples,
                 t_start):
        self.positions = np.asarray(positions, dtype=np.float64)
        self.sound_speed = sound_speed
        self.sample_rate = sample_rate
        self.n_samples = n_samples
        self.t_start = t_start

    @property
    def n_sensors(self):
        return self.positions.shape[0]


class Cloud:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _small_states(g):
    return oracle.States(g["small_a0"], g["small_p0"], g["small_mu"])


def test_forward_golden_small(golden):
    arr = small_array(golden, Arr)
    st = _small_states(golden)
    assert np.allclose(oracle.forward_frame(st, arr), golden["small_fwd"],
                       rtol=1e-12, atol=1e-15)
    assert np.allclose(oracle.forward_frame(st, arr, exact=True),
                       golden["small_fwd_exact"], rtol=1e-12, atol=1e-15)


def test_adjoint_golden_small(golden):
    arr = small_array(golden, Arr)
    st = _small_states(golden)
    G = oracle.frame_state_grads(st, arr, golden["small_res"])
    assert np.allclose(G, golden["small_G"], rtol=1e-11, atol=1e-16)
    G = oracle.frame_state_grads(st, arr, golden["small_res"], exact=True)
    assert np.allclose(G, golden["small_G_exact"], rtol=1e-11, atol=1e-16)


def test_planar_golden(golden):
    arr = planar_array(golden, Arr)
    st = oracle.States(golden["planar_a0"], golden["planar_p0"],
                       golden["planar_mu"])
    pred = oracle.forward_frame(st, arr)
    assert rel_l2(pred, golden["planar_pred"]) < 1e-13
    G = oracle.frame_state_grads(st, arr, golden["planar_res"])
    assert rel_l2(G, golden["planar_G"]) < 1e-12


@pytest.mark.parametrize("tag", ["sh", "pc"])
@pytest.mark.parametrize("mode", ["multiplicative", "additive", "radial"])
def test_deformation_golden(golden, tag, mode):
    g = golden
    cloud = Cloud(**{k: g[f"def_{tag}_{k}"] for k in
                     ("p0", "a0", "mu", "theta", "sigma", "omega")})
    key = f"def_{tag}_{mode[:3]}"
    st = oracle.cloud_states_at(cloud, 0.37, mode, a0_floor=0.3)
    assert np.allclose(st.a0_t, g[key + "_a0t"], rtol=1e-14, atol=0)
    assert np.allclose(st.p0_t, g[key + "_p0t"], rtol=1e-14, atol=0)
    assert np.allclose(st.mu_t, g[key + "_mut"], rtol=1e-14, atol=1e-15)
    jac = oracle.cloud_state_grads(cloud, 0.37, mode, a0_floor=0.3)
    for nm, arr in (("dbase", jac.d_base), ("domega", jac.d_omega),
                    ("dtheta", jac.d_theta), ("dsigma", jac.d_sigma)):
        assert np.allclose(arr, g[key + "_" + nm], rtol=1e-13, atol=1e-15)
    arr_ = small_array(golden, Arr)
    G = oracle.frame_state_grads(st, arr_, g[key + "_res"])
    cg = oracle.assemble_grads(G, jac)
    for nm in ("p0", "a0", "mu", "theta", "sigma", "omega"):
        assert np.allclose(getattr(cg, nm), g[key + "_g" + nm], rtol=1e-10,
                           atol=1e-14), nm


def test_adam_golden(golden):
    p = golden["adam_p0"].copy()
    st = oracle.Moments(np.zeros_like(p), np.zeros_like(p))
    for k in range(3):
        oracle.adam_step(p, golden["adam_g"][k], st, lr=1e-2 * (k + 1))
        assert np.array_equal(p, golden["adam_traj"][k])


def test_prune_golden(golden):
    keep = oracle.prune_keep(golden["prune_p0"], 1e-2)
    assert np.array_equal(keep.astype(np.uint8), golden["prune_keep"])
    idx = np.arange(len(keep))
    assert np.array_equal(oracle.compact(idx, keep), golden["prune_order"])


def test_dynamic_iterations_golden(golden):
    """Three full reference iterations (loop + Adam + floors)."""
    g = golden

    class Cfg:
        coord_mode = "multiplicative"
        a0_floor = 0.05
        sigma_floor = 1e-4
        p0_floor = 0.0
        support_sigmas = 6.0
        exact_forward = False

    B, nb = 4, 9
    th = np.arange(nb) / (nb - 1)
    cloud = Cloud(p0=g["dyn_p0"].copy(), a0=g["dyn_a0"].copy(),
                  mu=g["dyn_mu"].copy(),
                  theta=np.broadcast_to(th, (B, nb)).copy(),
                  sigma=np.full((B, nb), 2.0 / (nb - 1)),
                  omega=np.zeros((B, 5, nb)))
    arr = small_array(golden, Arr)
    data = g["dyn_data"]                       # (M, K, T)
    obs = np.transpose(data, (1, 0, 2))
    times = np.arange(3) / 2.0
    moments = {k: oracle.Moments(np.zeros_like(getattr(cloud, k)),
                                 np.zeros_like(getattr(cloud, k)))
               for k in ("p0", "a0", "mu", "theta", "sigma", "omega")}
    lrs = {"coords": 5e-3, "pressure": 2e-2, "std": 2e-3, "deform": 5e-3}
    losses = []
    for it in range(3):
        loss, grads = oracle.iteration_grads(cloud, times, obs, arr, Cfg)
        losses.append(loss)
        oracle.apply_step(cloud, grads, moments, lrs, Cfg)
    assert np.allclose(losses, g["dyn_loss"], rtol=1e-12)
    for nm in ("p0", "a0", "mu", "theta", "sigma", "omega"):
        assert np.allclose(getattr(cloud, nm), g["dyn_out_" + nm],
                           rtol=1e-12, atol=1e-15), nm


# ---- known-answer tests restated from the reference suite ---------------

def _one_ball_trace(R, a0, p0, v, t):
    """Closed form via the oracle with one ball on the x axis."""
    arr = Arr(np.array([[R, 0.0, 0.0]]), v, 1.0, 1, float(t))
    st = oracle.States(np.array([a0]), np.array([p0]), np.zeros((1, 3)))
    return oracle.forward_frame(st, arr, exact=True)[0, 0]


def test_peak_value_known_answer():
    """test_radiator.py:29-35: peak a0 e^{-1/2}/(2R) = 0.0025272110."""
    R, a0, v = 60.0, 0.5, 1.5
    got = _one_ball_trace(R, a0, 1.0, v, (R - a0) / v)
    assert got == pytest.approx(0.0025272110, rel=1e-6)


def test_initial_profile_known_answer():
    """test_radiator.py:22-27: t = 0 gives p0 exp(-R^2 / 2a0^2)."""
    for R, a0 in [(3.0, 1.0), (10.0, 2.5), (1.2, 0.7)]:
        got = _one_ball_trace(R, a0, 1.3, 1.5, 0.0)
        assert got == pytest.approx(1.3 * math.exp(-R * R / (2 * a0 * a0)),
                                    rel=1e-12)


def test_eval_basis_known_answer():
    """test_deformation.py:31-35: exp(-1/2) = 0.6065306597126334."""
    v, _, _ = oracle.gauss_pieces(0.6, 0.5, 0.1)
    assert v == pytest.approx(0.6065306597126334)


def test_identity_bit_exact():
    """test_deformation.py:86-93 / acceptance criterion 3."""
    rng = np.random.default_rng(3)
    B, nb = 7, 65
    th = np.arange(nb) / (nb - 1)
    cloud = Cloud(p0=rng.uniform(0.1, 2, B), a0=rng.uniform(0.1, 1, B),
                  mu=rng.uniform(-5, 5, (B, 3)),
                  theta=np.broadcast_to(th, (B, nb)).copy(),
                  sigma=np.full((B, nb), 2.0 / (nb - 1)),
                  omega=np.zeros((B, 5, nb)))
    for t in np.linspace(0, 1, 11):
        st = oracle.cloud_states_at(cloud, t)
        assert np.array_equal(st.a0_t, cloud.a0)
        assert np.array_equal(st.p0_t, cloud.p0)
        assert np.array_equal(st.mu_t, cloud.mu)


def test_l2_constant_offset():
    """test_reconstruction.py:25-27."""
    o = np.zeros((2, 4))
    assert oracle.l2_loss(o + 1.0, o) == 4.0


def test_adam_first_step_and_fixed_point():
    """test_reconstruction.py:53-64."""
    p = np.array([3.0])
    st = oracle.Moments(np.zeros(1), np.zeros(1))
    oracle.adam_step(p, np.array([1.0]), st, lr=0.1)
    assert p[0] == pytest.approx(2.9, abs=1e-6)
    p = np.array([1.5, -2.0])
    st = oracle.Moments(np.zeros(2), np.zeros(2))
    oracle.adam_step(p, np.zeros(2), st, lr=0.1)
    assert np.array_equal(p, [1.5, -2.0])
    with pytest.raises(ValueError, match="pressure"):
        oracle.adam_step(p, np.array([np.nan, 0]), st, 0.1, "pressure")


def test_schedule_boundaries():
    """test_reconstruction.py:45-49."""
    assert oracle.scheduled_lr(1.0, 159, 160, 0.1) == 1.0
    assert oracle.scheduled_lr(1.0, 160, 160, 0.1) == 0.1


def test_coincidence_message():
    arr = Arr(np.array([[1.0, 2.0, 3.0], [0.0, 0.0, 30.0]]), 1.5, 8.0, 64,
              14.0)
    st = oracle.States(np.array([0.5]), np.array([1.0]),
                       np.array([[0.0, 0.0, 30.0]]))
    with pytest.raises(ValueError, match=r"ball 0 .* sensor 1"):
        oracle.forward_frame(st, arr)


# ---- builder-defined (unpinned) rules: self-consistency only ------------

def test_polyfourier_basis_values():
    phi = oracle.polyfourier_basis(0.25, 2)
    assert phi.shape == (8,)
    assert np.allclose(phi[:4], [1, 0.25, 0.0625, 0.015625])
    assert np.allclose(phi[4:], [1.0, 0.0, 0.0, -1.0], atol=1e-15)


def test_densify_plan_order_and_percentile():
    rng = np.random.default_rng(0)
    p0 = rng.uniform(0, 0.05, 50)
    g = rng.normal(size=50)
    keep, split, index, child = oracle.densify_plan(p0, g)
    thr = np.percentile(np.abs(g), 90)
    assert np.array_equal(keep, ~(p0 < 0.01))
    assert np.array_equal(split, (np.abs(g) > thr) & keep)
    assert np.array_equal(index[:keep.sum()], np.nonzero(keep)[0])
    assert np.array_equal(index[keep.sum():], np.nonzero(split)[0])
    assert child.sum() == split.sum()


# ---- live reference (build container only) -------------------------------

@pytest.mark.reference
def test_oracle_matches_live_reference(ref_pkg):
    from pacloud.core import DynamicCloud
    from pacloud.deformation import CloudState, cloud_state_grads, \
        cloud_states_at
    from pacloud.geometry import spherical_array
    from pacloud.radiator import accumulate_frame_grads, forward_frame
    rng = np.random.default_rng(99)
    arr = spherical_array(12, 30.0, sample_rate=8.0, n_samples=96,
                          t_start=14.0)
    B, nb = 9, 4
    cloud = DynamicCloud(rng.uniform(0.3, 1, B), rng.uniform(0.3, 0.9, B),
                         rng.uniform(-4, 4, (B, 3)),
                         rng.uniform(0, 1, (B, 5, nb)),
                         rng.uniform(0.1, 0.5, (B, 5, nb)),
                         rng.uniform(-0.3, 0.3, (B, 5, nb)))
    for mode in ("multiplicative", "additive", "radial"):
        st_r = cloud_states_at(cloud, 0.42, mode, a0_floor=0.3)
        st_o = oracle.cloud_states_at(cloud, 0.42, mode, a0_floor=0.3)
        assert np.allclose(st_r.mu_t, st_o.mu_t, rtol=1e-14)
        pr = forward_frame(st_r, arr)
        po = oracle.forward_frame(st_o, arr)
        assert np.allclose(pr, po, rtol=1e-12, atol=1e-16)
        res = rng.normal(0, 1e-3, pr.shape)
        cr = accumulate_frame_grads(st_r, cloud_state_grads(
            cloud, 0.42, mode, a0_floor=0.3), arr, res)
        co = oracle.assemble_grads(oracle.frame_state_grads(st_o, arr, res),
                                   oracle.cloud_state_grads(
                                       cloud, 0.42, mode, a0_floor=0.3))
        for nm in ("p0", "a0", "mu", "theta", "sigma", "omega"):
            assert np.allclose(getattr(cr, nm), getattr(co, nm), rtol=1e-10,
                               atol=1e-15), (mode, nm)
