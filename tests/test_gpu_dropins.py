"""Drop-ins that round 1 left without a CUDA-path test: the formula anchors
(radiator.py:36-83), the single-ball deformation API (deformation.py:57-181),
the float64 drop-in deformation / optimiser numerics and the reference's
per-array guard order inside the deform group (reconstruction.py:88-93).

Each case restates a reference known answer (pkg/tests/test_radiator.py,
test_deformation.py) and runs it through the C ABI on the device."""

import math

import numpy as np
import pytest

import oracle
from helpers import rel_err

pytestmark = pytest.mark.gpu


# ------------------------------------------------- pressure_kernel (A11)

def test_pressure_zero_source(pc):
    """test_radiator.py:18-20."""
    t = np.linspace(0, 50, 100)
    assert np.all(pc.pressure_kernel(60.0, t, 0.0, 0.5, 1.5) == 0.0)


def test_pressure_initial_profile(pc):
    """test_radiator.py:22-27: both terms coincide at t = 0."""
    for R, a0 in [(3.0, 1.0), (10.0, 2.5), (1.2, 0.7)]:
        got = pc.pressure_kernel(R, 0.0, 1.3, a0, 1.5)
        assert got == pytest.approx(1.3 * math.exp(-R * R / (2 * a0 * a0)),
                                    rel=1e-12)


def test_pressure_peak_known_answer(pc):
    """test_radiator.py:29-35: a0 e^{-1/2} / (2R) = 0.0025272110."""
    R, a0, v = 60.0, 0.5, 1.5
    got = pc.pressure_kernel(R, (R - a0) / v, 1.0, a0, v)
    assert got == pytest.approx(a0 * math.exp(-0.5) / (2 * R), rel=1e-6)
    assert got == pytest.approx(0.0025272110, rel=1e-6)


def test_pressure_nonpositive_distance(pc):
    for R in (0.0, -2.0):
        with pytest.raises(ValueError):
            pc.pressure_kernel(R, 1.0, 1.0, 0.5, 1.5)


def test_pressure_antisymmetry(pc):
    """test_radiator.py:43-49."""
    R, a0, v = 60.0, 1.0, 1.5
    tau = np.linspace(0.01, 4 * a0 / v, 50)
    peak = a0 * math.exp(-0.5) / (2 * R)
    late = pc.pressure_kernel(R, R / v + tau, 1.0, a0, v)
    early = pc.pressure_kernel(R, R / v - tau, 1.0, a0, v)
    assert np.max(np.abs(late + early)) < 1e-6 * peak


def test_pressure_one_over_R(pc):
    """test_radiator.py:51-57."""
    a0, v = 0.8, 1.5
    off = np.linspace(-5 * a0, 5 * a0, 400)
    for R in (20.0, 45.0):
        near = pc.pressure_kernel(R, (R + off) / v, 1.0, a0, v)
        far = pc.pressure_kernel(2 * R, (2 * R + off) / v, 1.0, a0, v)
        assert np.max(near) == pytest.approx(2 * np.max(far), rel=1e-6)


def _spherical_mean(R, t, p0, a0, v, n_nodes=240, h_rel=5e-4):
    """Quadrature of the spherical-mean solution (the reference suite's
    oracle for the closed form, restated): p(R, t) = d/dt [t <f>_{S(vt)}]
    with f the Gaussian initial pressure; the sphere average by
    Gauss-Legendre over the polar cosine, restricted to where f is above
    ~1e-31 of its peak (12 a0), the time derivative by central
    differences."""
    nodes, weights = np.polynomial.legendre.leggauss(n_nodes)
    cut = 12.0 * a0

    def average(rho):
        rho = abs(rho)
        if rho == 0.0:
            return p0 * math.exp(-R * R / (2 * a0 * a0))
        if abs(R - rho) >= cut:
            return 0.0
        # |x - s|^2 = R^2 + rho^2 + 2 R rho u; keep u where |x - s| < cut
        s_hi = min(R + rho, cut)
        u_hi = min(1.0, max(-1.0, (s_hi * s_hi - R * R - rho * rho) /
                            (2 * R * rho)))
        half = 0.5 * (u_hi + 1.0)
        u = -1.0 + half * (nodes + 1.0)
        f = p0 * np.exp(-(R * R + rho * rho + 2 * R * rho * u) /
                        (2 * a0 * a0))
        return 0.5 * half * float(weights @ f)

    out = np.empty(len(t))
    for i, ti in enumerate(t):
        h = h_rel * a0 / v
        out[i] = ((ti + h) * average(v * (ti + h)) -
                  (ti - h) * average(v * (ti - h))) / (2 * h)
    return out


def test_pressure_quadrature_oracle(pc):
    """test_radiator.py:59-69: closed form vs the spherical-mean quadrature
    at rel-L2 < 1e-3."""
    rng = np.random.default_rng(3)
    for _ in range(5):
        R, a0, v = rng.uniform(10, 100), rng.uniform(0.2, 3.0), 1.5
        t = np.linspace(max(0.0, (R - 8 * a0) / v), (R + 8 * a0) / v, 160)
        mine = pc.pressure_kernel(R, t, 1.0, a0, v)
        ref = _spherical_mean(R, t, 1.0, a0, v)
        assert np.linalg.norm(mine - ref) / np.linalg.norm(ref) < 1e-3


def test_pressure_grad_linear_in_p0(pc):
    """test_radiator.py:73-77."""
    R, t, a0, v = 40.0, 26.0, 1.0, 1.5
    d_p0, _, _ = pc.pressure_kernel_grad(R, t, 1.0, a0, v)
    assert d_p0 == pytest.approx(pc.pressure_kernel(R, t, 1.0, a0, v),
                                 rel=1e-14)


def test_pressure_grad_flat_tail(pc):
    """test_radiator.py:79-82."""
    _, d_a0, _ = pc.pressure_kernel_grad(60.0, 0.0, 1.0, 0.5, 1.5)
    assert abs(d_a0) < 1e-300


def test_pressure_grad_finite_differences(pc):
    """test_radiator.py:84-106: (p0, a0, R) partials vs central differences
    at < 1e-4 (vectorised: one device call per perturbation)."""
    rng = np.random.default_rng(11)
    n = 200
    R = rng.uniform(10, 100, n)
    a0 = rng.uniform(0.2, 3.0, n)
    p0 = rng.uniform(0.1, 2.0, n)
    v = 1.5
    t = rng.uniform((R - 6 * a0) / v, (R + 6 * a0) / v)
    ana = np.stack(pc.pressure_kernel_grad(R, t, p0, a0, v))
    num = np.zeros_like(ana)
    args = {"p0": p0, "a0": a0, "R": R}
    for i, name in enumerate(("p0", "a0", "R")):
        h = 1e-6 * np.abs(args[name])
        hi, lo = dict(args), dict(args)
        hi[name] = args[name] + h
        lo[name] = args[name] - h
        num[i] = (pc.pressure_kernel(hi["R"], t, hi["p0"], hi["a0"], v) -
                  pc.pressure_kernel(lo["R"], t, lo["p0"], lo["a0"], v)) / (2 * h)
    worst = max(float(np.max(rel_err(ana[:, k], num[:, k], floor_rel=1e-6)))
                for k in range(n))
    assert worst < 1e-4


def test_forward_kernel_reproduces_pressure_kernel(pc):
    """The CUDA forward sweep (one ball, exact=True, every sample) against
    the closed form on the device: the formula anchor of radiator.py:36-55
    as the hot kernel evaluates it (fp32 samples, 1e-5 relative L2)."""
    R, a0, p0, v, fs, T = 30.0, 0.6, 0.8, 1.5, 40.0, 2048
    arr = pc.SensorArray(np.array([[R, 0.0, 0.0], [0.0, R * 0.9, 0.0]]),
                         v, fs, T, 0.0)
    st = pc.CloudState(np.array([a0]), np.array([p0]), np.zeros((1, 3)))
    out = pc.forward_frame(st, arr, exact=True)
    t = np.arange(T) / fs
    for m, Rm in enumerate((R, 0.9 * R)):
        want = pc.pressure_kernel(Rm, t, p0, a0, v)
        assert np.linalg.norm(out[m] - want) / np.linalg.norm(want) < 1e-5


def test_adjoint_kernel_reproduces_pressure_grad(pc):
    """The CUDA adjoint on one ball and a unit residual at one sample
    returns pressure_kernel_grad's (a0, p0, R) partials (chain to mu_x)."""
    R, a0, p0, v, fs, T = 30.0, 0.6, 0.8, 1.5, 40.0, 2048
    arr = pc.SensorArray(np.array([[R, 0.0, 0.0]]), v, fs, T, 0.0)
    st = pc.CloudState(np.array([a0]), np.array([p0]), np.zeros((1, 3)))
    j = int(round((R - 0.3 * a0) / v * fs))
    resid = np.zeros((1, T))
    resid[0, j] = 1.0
    G = pc.frame_state_grads(st, arr, resid, exact=True)[0]
    d_p0, d_a0, d_R = pc.pressure_kernel_grad(R, j / fs, p0, a0, v)
    # dR/dmu_x = (mu_x - s_x)/R = -1 for a sensor on +x
    want = np.array([d_a0, d_p0, -d_R, 0.0, 0.0])
    scale = np.max(np.abs(want))
    assert np.max(np.abs(G - want)) < 1e-4 * scale


# ---------------------------------------- single-ball deformation (A1/A2)

def test_eval_basis_known_answers(pc):
    """test_deformation.py:27-45."""
    assert pc.eval_basis(0.5, 0.5, 0.1) == 1.0
    assert pc.eval_basis(0.6, 0.5, 0.1) == pytest.approx(math.exp(-0.5),
                                                         rel=1e-12)
    assert pc.eval_basis(0.6, 0.5, 0.1) == pytest.approx(0.6065306597126334)
    assert pc.eval_basis(0.5, 0.0, 1e9) == pytest.approx(1.0, abs=1e-12)
    for s in (0.0, -1.0):
        with pytest.raises(ValueError):
            pc.eval_basis(0.5, 0.5, s)
    rng = np.random.default_rng(0)
    t, th, sg = rng.uniform(-2, 3, 500), rng.uniform(0, 1, 500), \
        rng.uniform(1e-3, 10, 500)
    v = pc.eval_basis(t, th, sg)
    assert np.all((v >= 0) & (v <= 1))
    live = 0.5 * ((t - th) / sg) ** 2 < 700.0
    assert np.all(v[live] > 0)
    assert np.allclose(v, np.exp(-0.5 * ((t - th) / sg) ** 2), rtol=1e-12,
                       atol=0)


def test_eval_H_known_answers(pc):
    """test_deformation.py:56-82."""
    from paper_2412_03898_b200.core import default_basis_grid
    th, sg = default_basis_grid(5)
    assert pc.eval_H(0.3, np.zeros(5), th, sg) == 0.0
    assert pc.eval_H(0.7, [0.3], [0.7], [0.2]) == pytest.approx(0.3)
    got = pc.eval_H(0.0, [0.5, -0.2], [0.0, 1.0], [1.0, 1.0])
    assert got == pytest.approx(0.5 - 0.2 * math.exp(-0.5), rel=1e-12)
    assert got == pytest.approx(0.37869386805747335)
    with pytest.raises(ValueError):
        pc.eval_H(0.0, [0.5, 0.2], [0.0], [1.0, 1.0])
    om = np.array([0.4, -0.1, 0.2])
    th3, sg3 = np.array([0.1, 0.5, 0.9]), np.array([0.2, 0.3, 0.1])
    h1 = pc.eval_H(0.4, om, th3, sg3)
    for scale in (-3.0, -0.7, 0.0, 1.3, 2.9):
        assert pc.eval_H(0.4, scale * om, th3, sg3) == \
            pytest.approx(scale * h1, rel=1e-12, abs=1e-15)


def test_ball_state_at_known_answers(pc):
    """test_deformation.py:86-140 (identity bit-exact with non-fp32 values,
    pressure substitution, mode semantics, floor, bad mode)."""
    from paper_2412_03898_b200.core import DeformField, GaussBall
    rng = np.random.default_rng(1234)
    ball = GaussBall(1.7, 0.31, rng.uniform(-5, 5, 3))
    ident = DeformField.identity(65)
    for t in np.linspace(0, 1, 11):
        s = pc.ball_state_at(ball, ident, t)
        assert s.a0_t == ball.a0 and s.p0_t == ball.p0
        assert np.array_equal(s.mu_t, ball.mu)
    om = np.zeros((5, 1))
    om[1, 0] = 0.1
    s = pc.ball_state_at(GaussBall(2.0, 1.0, (0, 0, 0)),
                         DeformField([0.5], [0.2], om), 0.5)
    assert s.p0_t == pytest.approx(2.2, rel=1e-12)
    om = np.zeros((5, 1))
    om[2, 0] = 0.25
    s = pc.ball_state_at(GaussBall(1.0, 1.0, (0, 0, 0)),
                         DeformField([0.5], [0.3], om), 0.5, "additive")
    assert s.mu_t[0] == pytest.approx(0.25) and s.mu_t[1] == 0.0
    om = np.zeros((5, 1))
    om[2, 0] = 0.5
    s = pc.ball_state_at(GaussBall(1.0, 1.0, (2.0, -1.0, 4.0)),
                         DeformField([0.5], [0.3], om), 0.5, "radial")
    assert np.allclose(s.mu_t, [3.0, -1.5, 6.0])
    om = np.zeros((5, 1))
    om[0, 0] = -0.999
    s = pc.ball_state_at(GaussBall(1.0, 1.0, (0, 0, 0)),
                         DeformField([0.5], [0.3], om), 0.5, a0_floor=0.05)
    assert s.a0_t == 0.05
    with pytest.raises(ValueError):
        pc.ball_state_at(GaussBall(1, 1, (0, 0, 0)), ident, 0.5, "spiral")


@pytest.mark.parametrize("mode", ["multiplicative", "additive", "radial"])
@pytest.mark.parametrize("shared", [True, False])
def test_ball_state_grad_vs_oracle(pc, mode, shared):
    """ball_state_grad = the one-ball Jacobian of the oracle restatement of
    deformation.py:153-181 (and its FD, test_deformation.py:240-254)."""
    from paper_2412_03898_b200.core import DeformField, GaussBall
    rng = np.random.default_rng(7)
    n = 6
    theta, sigma = rng.uniform(0, 1, n), rng.uniform(0.05, 0.5, n)
    omega = rng.uniform(-0.5, 0.5, (5, n))
    if not shared:
        theta = np.tile(theta, (5, 1)) + rng.uniform(-0.02, 0.02, (5, n))
        sigma = np.tile(sigma, (5, 1)) * rng.uniform(0.9, 1.1, (5, n))
    ball = GaussBall(1.3, 0.7, rng.uniform(-3, 3, 3))
    field = DeformField(theta, sigma, omega)
    t = 0.37
    g = pc.ball_state_grad(ball, field, t, mode)
    cloud = pc.DynamicCloud(np.array([ball.p0]), np.array([ball.a0]),
                            np.asarray(ball.mu)[None], theta[None],
                            sigma[None], omega[None])
    ref = oracle.cloud_state_grads(cloud, t, mode)
    assert np.allclose(g.d_base, ref.d_base[0], rtol=1e-12, atol=1e-14)
    assert np.allclose(g.d_omega, ref.d_omega[0], rtol=1e-12, atol=1e-14)
    s0 = pc.ball_state_at(ball, field, t, mode)
    st = oracle.cloud_states_at(cloud, t, mode)
    assert s0.a0_t == pytest.approx(float(st.a0_t[0]), rel=1e-14)
    assert np.allclose(s0.mu_t, st.mu_t[0], rtol=1e-14, atol=1e-14)


def test_cloud_states_at_float64_identity(pc):
    """the drop-in returns float64 a0_t / p0_t; the identity
    deformation is bit-exact on values that are not fp32-representable
    (a0 = 0.31, p0 = 1.7, deformation.py:119-121)."""
    from paper_2412_03898_b200.core import default_basis_grid
    B, N = 7, 65
    th, sg = default_basis_grid(N)
    rng = np.random.default_rng(2)
    cloud = pc.DynamicCloud(np.full(B, 1.7), np.full(B, 0.31),
                            rng.uniform(-5, 5, (B, 3)), np.tile(th, (B, 1)),
                            np.tile(sg, (B, 1)), np.zeros((B, 5, N)))
    for mode in ("multiplicative", "additive", "radial"):
        for t in (0.0, 0.45, 1.0):
            s = pc.cloud_states_at(cloud, t, mode)
            assert s.a0_t.dtype == np.float64
            assert np.array_equal(s.a0_t, cloud.a0)
            assert np.array_equal(s.p0_t, cloud.p0)
            assert np.array_equal(s.mu_t, cloud.mu)


def test_cloud_states_at_floor_semantics(pc):
    """deformation.py:202-203: the floor applies whenever it is not None,
    including a0_floor <= 0."""
    from paper_2412_03898_b200.core import default_basis_grid
    B, N = 4, 3
    th, sg = default_basis_grid(N)
    om = np.zeros((B, 5, N))
    om[:, 0, :] = -0.9
    cloud = pc.DynamicCloud(np.ones(B), np.ones(B), np.ones((B, 3)),
                            np.tile(th, (B, 1)), np.tile(sg, (B, 1)), om)
    ref_none = oracle.cloud_states_at(cloud, 0.5)
    assert np.all(ref_none.a0_t < -1.4)            # a0 (1 + H0) < 0 here
    got = pc.cloud_states_at(cloud, 0.5)           # no floor: unclamped
    assert np.allclose(got.a0_t, ref_none.a0_t, rtol=1e-14)
    for floor in (-2.0, -1.0, 0.0, 0.5):
        got = pc.cloud_states_at(cloud, 0.5, a0_floor=floor)
        assert np.allclose(got.a0_t, np.maximum(ref_none.a0_t, floor),
                           rtol=1e-14), floor


# ------------------------------------------------ optimiser drop-ins (A8)

def test_adam_step_float64_matches_oracle(pc):
    """reconstruction.py:57-69 in float64: a finite gradient
    beyond the fp32 range is stepped, not rejected; values to 1e-15."""
    from paper_2412_03898_b200.reconstruction import AdamState
    rng = np.random.default_rng(4)
    p = rng.normal(size=50)
    g = rng.normal(size=50) * 1e-3
    g[3] = 1e39                                   # finite in fp64 only
    st = AdamState(np.zeros(50), np.zeros(50), 0)
    ref_p = p.copy()
    ref_st = oracle.Moments(np.zeros(50), np.zeros(50), 0)
    for lr in (1e-2, 3e-3):
        pc.adam_step(p, g, st, lr, "pressure")
        oracle.adam_step(ref_p, g, ref_st, lr, "pressure")
    assert st.t == 2
    assert np.allclose(p, ref_p, rtol=1e-14, atol=1e-16)
    assert np.allclose(st.m, ref_st.m, rtol=1e-14, atol=1e-16)


def test_sgd_step_float64(pc):
    p = np.array([1.0, 2.0, 3.0]) + 1e-12
    pc.sgd_step(p, np.array([0.5, -1.0, 1e39]), 1e-40, "coords")
    assert np.array_equal(p, np.array([1.0, 2.0, 3.0]) + 1e-12 -
                          1e-40 * np.array([0.5, -1.0, 1e39]))
    with pytest.raises(ValueError, match="coords"):
        pc.sgd_step(p, np.array([np.inf, 0.0, 0.0]), 0.1, "coords")


# -------------------- guard order inside the deform group (A8)

def test_engine_nan_in_omega_steps_theta_sigma_first(pc):
    """reconstruction.py:88-93, 320-327: the deform group steps theta, then
    sigma, then omega, one array at a time; a non-finite omega gradient
    raises naming 'deform' after theta and sigma have been updated (and
    their step counts advanced), omega untouched."""
    from paper_2412_03898_b200 import synth
    from paper_2412_03898_b200.core import DynamicCloud, ReconConfig
    from paper_2412_03898_b200.engine import IterationEngine
    prob = synth.make_problem(2, n_balls=200, n_sensors=32, n_frames=3)
    B, nb = 200, 5
    rng = np.random.default_rng(9)
    c = prob.cloud
    theta = np.tile(np.linspace(0, 1, nb), (B, 1))
    sigma = np.full((B, nb), 0.3)
    omega = rng.uniform(-0.02, 0.02, (B, 5, nb))
    prob.cloud = DynamicCloud(c.p0, c.a0, c.mu, theta, sigma, omega)
    prob.config = ReconConfig(n_basis=nb)
    obs = np.stack([oracle.forward_frame(oracle.States(a, p, m), prob.array)
                    for a, p, m in prob.gt_frames]).astype(np.float32)
    eng = IterationEngine(prob.cloud, prob.array, obs, prob.frame_times,
                          prob.config)
    eng.iterate(0, np.arange(prob.n_frames))
    seg = eng.layout.by_name
    before = {k: eng.P[s.offset:s.offset + s.size].clone()
              for k, s in seg.items()}
    steps = dict(eng.step_count)
    orig = eng.allreduce

    def poison():
        orig()
        eng.Gf[seg["omega"].offset + 11] = float("nan")
    eng.allreduce = poison
    with pytest.raises(ValueError, match="deform"):
        eng.iterate(1, np.arange(prob.n_frames))
    for k, s in seg.items():
        after = eng.P[s.offset:s.offset + s.size]
        changed = not bool((after == before[k]).all())
        if k == "omega":
            assert not changed and eng.step_count[k] == steps[k]
        else:
            assert changed, k
            assert eng.step_count[k] == steps[k] + 1, k


def test_validate_cloud(pc):
    """core.py:271-292 (test_core.py:83-112)."""
    from paper_2412_03898_b200.core import Box, default_basis_grid
    th, sg = default_basis_grid(3)
    B = 4
    cloud = pc.DynamicCloud(np.ones(B), np.ones(B), np.zeros((B, 3)),
                            np.tile(th, (B, 1)), np.tile(sg, (B, 1)),
                            np.zeros((B, 5, 3)))
    assert pc.validate_cloud(cloud, Box.cube(5.0)) == []
    cloud.a0[1] = 0.0
    cloud.p0[2] = -1.0
    cloud.mu[3] = (9.0, 0.0, 0.0)
    cloud.sigma[0, 1] = 0.0
    v = pc.validate_cloud(cloud, Box.cube(5.0))
    assert {(x.index, x.field) for x in v} == \
        {(1, "a0"), (2, "p0"), (3, "mu"), (0, "sigma")}
