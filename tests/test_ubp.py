"""universal back-projection against the live
reference's golden run and the C oracle."""

import numpy as np
import pytest

import oracle
from helpers import rel_l2
from paper_2412_03898_b200.core import SensorArray


def _case(golden):
    from paper_2412_03898_b200.evaluation import GridSpec
    c = golden["ubp_cfg"]
    arr = SensorArray(golden["ubp_pos"], c[0], c[1], int(c[2]), c[3])
    s = golden["ubp_spec"]
    return arr, GridSpec(s[:3], s[3], tuple(int(d) for d in s[4:7]))


def test_oracle_ubp_golden(golden):
    arr, spec = _case(golden)
    got = oracle.ubp_reconstruct(golden["ubp_traces"], arr, spec.origin,
                                 spec.spacing, spec.dims)
    assert np.allclose(got, golden["ubp_grid"], rtol=1e-10, atol=1e-14)


def test_compute_time_window_golden(golden):
    from paper_2412_03898_b200.core import Box
    from paper_2412_03898_b200.geometry import spherical_array
    from paper_2412_03898_b200.radiator import compute_time_window
    arr = spherical_array(48, 25.0, sample_rate=8.0)
    t0, n = compute_time_window(arr, Box.cube(4.0), 1.0)
    c = golden["ubp_cfg"]
    assert t0 == c[3] and n == int(c[2])
    with pytest.raises(ValueError):
        compute_time_window(arr, Box.cube(30.0), 1.0)
    with pytest.raises(ValueError):
        compute_time_window(arr, Box.cube(4.0), -1.0)


@pytest.mark.gpu
def test_ubp_kernel_golden(pc, golden):
    from paper_2412_03898_b200.ubp import ubp_reconstruct
    arr, spec = _case(golden)
    got = ubp_reconstruct(golden["ubp_traces"], arr, spec)
    want = golden["ubp_grid"]
    assert rel_l2(got.values, want) < 1e-5
    assert np.abs(got.values - want).max() < 1e-5 * np.abs(want).max()


@pytest.mark.gpu
def test_ubp_kernel_vs_oracle_large(pc, golden):
    """More sensors than one shared-memory chunk, dims not multiples of the
    tile, odd T (scalar filter edges)."""
    from paper_2412_03898_b200.evaluation import GridSpec
    from paper_2412_03898_b200.geometry import spherical_array
    from paper_2412_03898_b200.ubp import ubp_reconstruct
    arr = spherical_array(300, 20.0, sample_rate=10.0).with_window(5.0, 333)
    rng = np.random.default_rng(8)
    tr = rng.normal(size=(300, 333))
    spec = GridSpec(np.array([-3.0, -2.7, -3.1]), 0.31, (13, 19, 21))
    got = ubp_reconstruct(tr, arr, spec).values
    want = oracle.ubp_reconstruct(tr, arr, spec.origin, spec.spacing,
                                  spec.dims)
    assert rel_l2(got, want) < 1e-5


@pytest.mark.gpu
def test_ubp_errors(pc, golden):
    from paper_2412_03898_b200.evaluation import GridSpec
    from paper_2412_03898_b200.ubp import ubp_reconstruct
    arr, spec = _case(golden)
    with pytest.raises(ValueError, match="does not match"):
        ubp_reconstruct(golden["ubp_traces"][:, :10], arr, spec)
    short = arr.with_window(arr.t_start + 5.0, arr.n_samples)
    with pytest.raises(ValueError, match="sample window"):
        ubp_reconstruct(golden["ubp_traces"], short, spec)
    big = GridSpec(spec.origin * 20, spec.spacing * 20, spec.dims)
    with pytest.raises(ValueError, match="sample window"):
        ubp_reconstruct(golden["ubp_traces"], arr, big)
