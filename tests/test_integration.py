"""INTEGRATION.md made executable.

* section 2 (raw ctypes binding): the documented `PcArray` is extracted from
  the markdown and must have the layout of `_lib.PcArray` /
  include/pacloud_b200.h `pc_array_t` (CPU); on the GPU the documented
  `forward_traces` runs and matches the oracle.
* section 1 (patching the reference): `integration.enable()` is applied to
  the INSTALLED reference (`baseline/_ref/pacloud`, the reference arm's
  `pip install --target`), whose own `simulate_dataset` and
  `dynamic_reconstruct` then run through the patched names and are compared
  with the same functions unpatched (numba, fp64).  The import-time
  bindings patched are reconstruction.py:18-21, geometry.py:16-17 and
  cli.py:18-25.
"""

import ctypes
import re
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
from helpers import GRAD_TOL, SIGNAL_TOL, rel_l2

ROOT = Path(__file__).resolve().parents[1]
REF_INSTALL = ROOT / "baseline" / "_ref"


def _doc_block(section: str) -> str:
    """The first ```python block after the heading that starts `section`."""
    text = (ROOT / "INTEGRATION.md").read_text()
    start = text.index(section)
    m = re.search(r"```python\n(.*?)```", text[start:], re.S)
    return m.group(1)


def _doc_namespace():
    code = _doc_block("## 2. Raw C ABI via ctypes")
    code = code.replace('ctypes.CDLL("paper_2412_03898_b200/libpacloud_b200.so")',
                        f'ctypes.CDLL("{ROOT}/paper_2412_03898_b200/libpacloud_b200.so")')
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md#2", "exec"), ns)
    return ns


def test_doc_pcarray_layout_matches_header():
    from paper_2412_03898_b200 import _lib
    doc = _doc_namespace()["PcArray"]
    # pc_array_t: ptr, 2 x i32, 4 x f64, 2 x i32, ptr, 2 x i32 = 72 bytes
    assert ctypes.sizeof(doc) == ctypes.sizeof(_lib.PcArray) == 72
    want = [(n, getattr(_lib.PcArray, n).offset) for n, _ in _lib.PcArray._fields_]
    got = [(n, getattr(doc, n).offset) for n, _ in doc._fields_]
    assert got == want


def _reference():
    """The installed reference package (baseline/_ref), or the one this
    process already imported."""
    if "pacloud" not in sys.modules:
        if not (REF_INSTALL / "pacloud").exists():
            pytest.skip("reference not installed in baseline/_ref")
        sys.path.insert(0, str(REF_INSTALL))
    import pacloud
    return pacloud


def test_enable_patches_import_time_bindings():
    """enable() reaches every module that bound a hot-path name at import,
    disable() restores the reference's functions (no compute: CPU)."""
    ref = _reference()
    import pacloud.geometry
    import pacloud.reconstruction
    import paper_2412_03898_b200 as b200
    from paper_2412_03898_b200 import integration
    orig = (pacloud.reconstruction.forward_frame,
            pacloud.geometry.forward_frame,
            pacloud.reconstruction.dynamic_reconstruct)
    try:
        done = integration.enable(level="calls")
        assert "reconstruction.forward_frame" in done
        assert "geometry.forward_frame" in done
        assert "reconstruction.adam_step" in done
        assert pacloud.reconstruction.forward_frame is b200.forward_frame
        assert pacloud.geometry.forward_frame is b200.forward_frame
        assert ref.forward_frame is b200.forward_frame
        assert pacloud.reconstruction.dynamic_reconstruct is orig[2]
        integration.enable()
        assert pacloud.reconstruction.dynamic_reconstruct is \
            b200.dynamic_reconstruct
        assert pacloud.geometry.simulate_dataset is b200.simulate_dataset
    finally:
        integration.disable()
    assert (pacloud.reconstruction.forward_frame,
            pacloud.geometry.forward_frame,
            pacloud.reconstruction.dynamic_reconstruct) == orig


# ------------------------------------------------------------------ GPU

def _scene(ref):
    """A small 3-frame scene in the reference's own types."""
    rng = np.random.default_rng(21)
    B, M, T, K = 40, 24, 1024, 3
    pos = ref.fibonacci_sphere(2 * M, 12.0)[:M]
    arr = ref.SensorArray(pos, 1.5, 40.0, T, 0.0)
    mu = rng.uniform(-3, 3, (B, 3))
    p0 = rng.uniform(0.3, 1.0, B)
    a0 = rng.uniform(0.3, 0.6, B)
    frames = []
    for k in range(K):
        s = 1.0 + 0.05 * np.sin(2 * np.pi * k / K)
        frames.append(ref.CloudState(a0 * s, p0, mu * s))
    init = [ref.GaussBall(float(p0[i] * 1.1), float(a0[i]),
                          mu[i] + rng.normal(0, 0.05, 3)) for i in range(B)]
    return arr, frames, init


@pytest.mark.gpu
def test_doc_ctypes_forward_matches_oracle():
    import torch
    ns = _doc_namespace()
    rng = np.random.default_rng(3)
    B, M, T = 300, 16, 2048
    pos = rng.normal(size=(M, 3))
    pos = 30.0 * pos / np.linalg.norm(pos, axis=1, keepdims=True)
    mu = rng.uniform(-5, 5, (B, 3))
    a0 = rng.uniform(0.2, 0.6, B).astype(np.float32)
    p0 = rng.uniform(0.1, 1.0, B).astype(np.float32)
    d = torch.device("cuda")
    out, flag = ns["forward_traces"](
        torch.as_tensor(mu, device=d).view(1, B, 3),
        torch.as_tensor(a0, device=d).view(1, B),
        torch.as_tensor(p0, device=d).view(1, B),
        torch.as_tensor(pos, device=d), 1.5, 0.0, 1 / 40.0, T, 6.0, False)
    torch.cuda.synchronize()
    assert int(flag.item()) == 2 ** 63 - 1

    class Arr:
        positions, sound_speed, sample_rate, n_samples, t_start = \
            pos, 1.5, 40.0, T, 0.0
    want = oracle.forward_frame(oracle.States(a0.astype(float),
                                              p0.astype(float), mu), Arr)
    assert rel_l2(out[0].double().cpu().numpy(), want) < SIGNAL_TOL


@pytest.mark.gpu
def test_reference_simulate_dataset_patched():
    ref = _reference()
    from paper_2412_03898_b200 import integration
    arr, frames, _ = _scene(ref)
    want = ref.simulate_dataset(frames, arr, noise_std=1e-4, seed=9)
    try:
        integration.enable()
        got = ref.simulate_dataset(frames, arr, noise_std=1e-4, seed=9)
        import pacloud.geometry
        got_mod = pacloud.geometry.simulate_dataset(frames, arr,
                                                    noise_std=1e-4, seed=9)
    finally:
        integration.disable()
    assert np.asarray(got.data).shape == np.asarray(want.data).shape
    assert rel_l2(got.data, want.data) < SIGNAL_TOL
    assert rel_l2(got_mod.data, want.data) < SIGNAL_TOL
    assert np.array_equal(got.frame_times, want.frame_times)


@pytest.mark.gpu
@pytest.mark.parametrize("level", ["calls", "stages"])
def test_reference_dynamic_reconstruct_patched(level):
    """The reference's dynamic_reconstruct: unpatched (numba, fp64) vs
    patched at `level` ("calls": the reference's own frame loop over the
    CUDA drop-ins; "stages": the fused engine)."""
    ref = _reference()
    import pacloud.reconstruction as rr
    from paper_2412_03898_b200 import integration
    arr, frames, init = _scene(ref)
    obs = ref.simulate_dataset(frames, arr)
    cfg = ref.ReconConfig(lr_coords=5e-3, lr_pressure=2e-2, lr_std=2e-3,
                          lr_deform=5e-3, dynamic_iters=3, n_basis=9, seed=2)
    log_ref, log_got = [], []
    want = rr.dynamic_reconstruct(obs, arr, init, cfg, progress=log_ref.append)
    try:
        integration.enable(level=level)
        got = rr.dynamic_reconstruct(obs, arr, init, cfg,
                                     progress=log_got.append)
    finally:
        integration.disable()
    l_ref = [r["loss"] for r in log_ref]
    l_got = [r["loss"] for r in log_got]
    assert rel_l2(l_got, l_ref) < SIGNAL_TOL
    for nm in ("p0", "a0", "mu", "theta", "sigma"):
        assert rel_l2(getattr(got, nm), getattr(want, nm)) < 1e-6, nm
    # omega starts at 0 and takes three sign-like Adam steps: compare the
    # updates themselves
    assert rel_l2(got.omega, want.omega) < 1e-3


@pytest.mark.gpu
def test_reference_frame_gradients_patched():
    """One frame of the reference's loop body (reconstruction.py:303-316)
    unpatched vs through the patched names: gradients within 1e-4."""
    ref = _reference()
    import pacloud.reconstruction as rr
    from paper_2412_03898_b200 import integration
    arr, frames, init = _scene(ref)
    obs = ref.simulate_dataset(frames, arr)
    B, nb = len(init), 9
    rng = np.random.default_rng(4)
    th, sg = ref.default_basis_grid(nb) if hasattr(ref, "default_basis_grid") \
        else rr.default_basis_grid(nb)
    cloud = ref.DynamicCloud(np.array([b.p0 for b in init]),
                             np.array([b.a0 for b in init]),
                             np.array([b.mu for b in init]),
                             np.tile(th, (B, 1)), np.tile(sg, (B, 1)),
                             rng.uniform(-0.05, 0.05, (B, 5, nb)))

    def grads():
        t = float(obs.frame_times[1])
        st = rr.cloud_states_at(cloud, t, "multiplicative", a0_floor=0.05)
        sgr = rr.cloud_state_grads(cloud, t, "multiplicative", a0_floor=0.05)
        pred = rr.forward_frame(st, arr)
        res = pred - obs.frame(1)
        g = rr.accumulate_frame_grads(st, sgr, arr, res)
        return pred, np.concatenate([np.ravel(getattr(g, k)) for k in
                                     ("p0", "a0", "mu", "theta", "sigma",
                                      "omega")])
    pred_ref, g_ref = grads()
    try:
        integration.enable(level="calls")
        pred, g = grads()
    finally:
        integration.disable()
    assert rel_l2(pred, pred_ref) < SIGNAL_TOL
    assert rel_l2(g, g_ref) < GRAD_TOL
