"""phantoms / arrays / simulate_dataset and
voxelize / MAP / SSIM, against golden vectors from the live reference
(tests/golden/make_golden.py, geometry_and_evaluation) and the C oracle."""

import numpy as np
import pytest

import oracle
from helpers import rel_l2
from paper_2412_03898_b200.core import Box, CloudState, SensorArray
from paper_2412_03898_b200.geometry import (PhantomSpec, box_lattice,
                                            build_phantom, fibonacci_sphere,
                                            pulsation_schedule)


def _specs():
    return {
        "heart": PhantomSpec("heart", Box.cube(12.0), n_frames=3, pitch=1.6,
                             voxel_pitch=1.0),
        "vasc": PhantomSpec("vascular", Box.cube(14.0), n_frames=3,
                            tree_depth=4, seed=3, voxel_pitch=1.0),
        "custom": PhantomSpec("custom", Box.cube(5.0), n_frames=4,
                              pulsation=0.2, voxel_pitch=0.5,
                              custom_balls=((1.0, 0.6, 0.0, 0.0, 0.0),
                                            (0.5, 0.4, 1.5, -1.0, 2.0))),
    }


def _small_array(golden):
    cfg = golden["small_cfg"]
    return SensorArray(golden["small_pos"], cfg[0], cfg[1], int(cfg[2]), cfg[3])


def _grid_spec(vec):
    from paper_2412_03898_b200.evaluation import GridSpec
    return GridSpec(vec[:3], vec[3], tuple(int(d) for d in vec[4:7]))


# ------------------------------------------------------------------ CPU

def test_fibonacci_sphere_golden(golden):
    assert np.array_equal(fibonacci_sphere(37, 12.5), golden["geo_fib"])
    with pytest.raises(ValueError):
        fibonacci_sphere(0, 1.0)
    with pytest.raises(ValueError):
        fibonacci_sphere(4, 0.0)


@pytest.mark.parametrize("name", ["heart", "vasc", "custom"])
def test_phantom_frames_bit_exact(golden, name):
    ph = build_phantom(_specs()[name], grids=False)
    for key, attr in (("a0", "a0_t"), ("p0", "p0_t"), ("mu", "mu_t")):
        got = np.stack([getattr(f, attr) for f in ph.frames])
        assert np.array_equal(got, golden[f"ph_{name}_{key}"]), key
    assert ph.n_frames == _specs()[name].n_frames
    assert len(ph.frame_times) == ph.n_frames


def test_phantom_spec_validation():
    with pytest.raises(ValueError):
        PhantomSpec("torus", Box.cube(5.0))
    with pytest.raises(ValueError):
        PhantomSpec("heart", Box.cube(5.0), n_frames=0)
    with pytest.raises(ValueError):
        build_phantom(PhantomSpec("heart", Box.cube(3.0)), grids=False)
    with pytest.raises(ValueError):
        build_phantom(PhantomSpec("custom", Box.cube(1.0),
                                  custom_balls=((1, 1, 5, 0, 0),)),
                      grids=False)


def test_lattice_and_schedule():
    pts = box_lattice(Box((0, 0, 0), (1.0, 2.0, 0.1)), 0.5)
    assert pts.shape == (2 * 4 * 1, 3)
    assert np.allclose(pulsation_schedule(5, 0.3)[[0, 2, 4]], 1.0)


def test_oracle_voxelize_golden(golden):
    spec = golden["vox_spec"]
    for key, exact in (("vox_fast", False), ("vox_exact", True)):
        got = oracle.voxelize(golden["vox_mu"], golden["vox_a0"],
                              golden["vox_p0"], spec[:3], spec[3],
                              spec[4:7].astype(int), exact=exact)
        assert np.allclose(got, golden[key], rtol=1e-12, atol=1e-300), key


def test_oracle_ssim_golden(golden):
    spec = golden["vox_spec"]
    st = (golden["vox_mu"], golden["vox_a0"], golden["vox_p0"])
    a = oracle.voxelize(*st, spec[:3], spec[3], spec[4:7].astype(int))
    b = oracle.voxelize(st[0] + 0.2, st[1] * 1.1, st[2], spec[:3], spec[3],
                        spec[4:7].astype(int))
    vals = []
    for ax, drop in (("XY", 2), ("YZ", 0), ("XZ", 1)):
        ma, mb = a.max(axis=drop), b.max(axis=drop)
        assert np.allclose(mb, golden[f"map_{ax}"], rtol=1e-12)
        peak = max(ma.max(), mb.max())
        vals.append(oracle.ssim(ma / peak, mb / peak))
    assert np.allclose(vals, golden["ssim_vals"], rtol=1e-12)


def test_ssim_host_identity_and_errors():
    from paper_2412_03898_b200.evaluation import ssim
    img = np.random.default_rng(0).uniform(size=(16, 20))
    assert ssim(img, img) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(ValueError):
        ssim(img, img[:, :19])
    with pytest.raises(ValueError):
        ssim(img[:10], img[:10])


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_voxelize_kernel_golden(pc, golden):
    from paper_2412_03898_b200.evaluation import voxelize
    spec = _grid_spec(golden["vox_spec"])
    st = CloudState(golden["vox_a0"], golden["vox_p0"], golden["vox_mu"])
    for key, exact in (("vox_fast", False), ("vox_exact", True)):
        got = voxelize(st, spec, exact=exact).values
        assert rel_l2(got, golden[key]) < 1e-6, key
        assert np.abs(got - golden[key]).max() < 1e-6 * golden[key].max()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["heart", "vasc", "custom"])
def test_phantom_grids_golden(pc, golden, name):
    ph = build_phantom(_specs()[name])
    want = golden[f"ph_{name}_grid0"]
    got = ph.grids[0]
    assert np.allclose(np.concatenate([got.origin, [got.spacing], got.dims]),
                       golden[f"ph_{name}_gridspec"])
    assert rel_l2(got.values, want) < 1e-6


@pytest.mark.gpu
def test_voxelize_kernel_vs_oracle_random(pc):
    """Larger random cloud, grid not a multiple of the 8^3 tile, balls
    partly outside the grid."""
    from paper_2412_03898_b200.evaluation import GridSpec, voxelize
    rng = np.random.default_rng(5)
    B = 3000
    mu = rng.uniform(-9, 9, (B, 3))
    a0 = rng.uniform(0.15, 0.9, B)
    p0 = rng.uniform(0.1, 1.0, B)
    spec = GridSpec(np.array([-8.0, -7.3, -8.1]), 0.27, (61, 57, 66))
    got = voxelize(CloudState(a0, p0, mu), spec).values
    want = oracle.voxelize(mu, a0, p0, spec.origin, spec.spacing, spec.dims)
    assert rel_l2(got, want) < 1e-6
    assert np.abs(got - want).max() < 2e-6 * want.max()


@pytest.mark.gpu
def test_voxelize_edges(pc):
    from paper_2412_03898_b200.evaluation import GridSpec, voxelize
    spec = GridSpec(np.zeros(3), 0.5, (1, 1, 1))
    empty = CloudState(np.zeros(0), np.zeros(0), np.zeros((0, 3)))
    assert voxelize(empty, spec).values.shape == (1, 1, 1)
    assert voxelize(empty, spec).values[0, 0, 0] == 0.0
    one = CloudState(np.array([0.5]), np.array([2.0]), np.zeros((1, 3)))
    assert voxelize(one, spec).values[0, 0, 0] == pytest.approx(2.0, rel=1e-6)
    with pytest.raises(ValueError):
        voxelize(CloudState(np.array([0.0]), np.array([1.0]),
                            np.zeros((1, 3))), spec)


@pytest.mark.gpu
def test_simulate_dataset_golden(pc, golden):
    """Batched GPU forward over all frames + the reference's noise draw."""
    from paper_2412_03898_b200.geometry import simulate_dataset
    ph = build_phantom(_specs()["custom"], grids=False)
    sig = simulate_dataset(ph, _small_array(golden), noise_std=1e-3, seed=7)
    want = golden["sim_data"]
    assert sig.data.shape == want.shape
    assert np.abs(sig.data - want).max() < 1e-5 * np.abs(want).max()
    assert np.allclose(sig.frame_times, np.linspace(0, 1, ph.n_frames))
    with pytest.raises(ValueError):
        simulate_dataset([], _small_array(golden))
    with pytest.raises(ValueError):
        simulate_dataset(ph, _small_array(golden), noise_std=-1.0)


@pytest.mark.gpu
def test_simulate_dataset_matches_oracle_forward(pc, golden):
    from paper_2412_03898_b200.geometry import simulate_dataset
    ph = build_phantom(_specs()["heart"], grids=False)
    arr = _small_array(golden)
    sig = simulate_dataset(ph, arr)
    for k, f in enumerate(ph.frames):
        want = oracle.forward_frame(oracle.States(f.a0_t, f.p0_t, f.mu_t), arr)
        assert rel_l2(sig.data[:, k, :], want) < 1e-5


@pytest.mark.gpu
def test_map_and_ssim_device_golden(pc, golden):
    from paper_2412_03898_b200.evaluation import (map_project, normalize_pair,
                                                  ssim, voxelize)
    spec = _grid_spec(golden["vox_spec"])
    st = CloudState(golden["vox_a0"], golden["vox_p0"], golden["vox_mu"])
    st2 = CloudState(st.a0_t * 1.1, st.p0_t, st.mu_t + 0.2)
    a, b = voxelize(st, spec), voxelize(st2, spec)
    for k, ax in enumerate(("XY", "YZ", "XZ")):
        mb = map_project(b, ax)
        assert rel_l2(mb.values, golden[f"map_{ax}"]) < 1e-6
        x, y = normalize_pair(map_project(a, ax), mb)
        assert ssim(x, y) == pytest.approx(golden["ssim_vals"][k], abs=1e-5)
