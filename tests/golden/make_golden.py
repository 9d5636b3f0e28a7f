"""Generate the golden vectors that pin the CPU oracle to the reference.

Run in the build container, where the read-only reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the UNMODIFIED reference package from /root/reference/pkg/src,
feeds it seeded float32-quantised inputs and stores inputs + outputs as
float64 in tests/golden/golden.npz.  The GPU box never needs /root/reference:
tests read only the .npz.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("PACLOUD_REF", "/root/reference/pkg/src"))
OUT = Path(__file__).with_name("golden.npz")


def q32(x):
    """Quantise to float32 and back (inputs identical on CPU and GPU)."""
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def main():
    sys.path.insert(0, str(REF))
    from pacloud.core import DynamicCloud, GaussBall, ReconConfig, \
        SensorArray, SignalSet, frame_times
    from pacloud.deformation import CloudState, cloud_state_grads, \
        cloud_states_at
    from pacloud.geometry import spherical_array
    from pacloud.radiator import accumulate_frame_grads, forward_frame, \
        frame_state_grads
    from pacloud.reconstruction import AdamState, adam_step, \
        dynamic_reconstruct

    g = {}
    rng = np.random.default_rng(20241205)

    # --- (1) small sphere array (reference conftest.small_array) ----------
    pos = q32(spherical_array(8, 30.0).positions)
    small = SensorArray(pos, 1.5, 8.0, 64, 14.0)
    B = 5
    st = CloudState(q32(rng.uniform(0.3, 1, B)), q32(rng.uniform(0.2, 1, B)),
                    q32(rng.uniform(-4, 4, (B, 3))))
    g["small_pos"] = pos
    g["small_cfg"] = np.array([1.5, 8.0, 64, 14.0])
    g["small_a0"], g["small_p0"], g["small_mu"] = st.a0_t, st.p0_t, st.mu_t
    g["small_fwd"] = forward_frame(st, small)
    g["small_fwd_exact"] = forward_frame(st, small, exact=True)
    res = q32(rng.normal(0, 1e-3, (8, 64)))
    g["small_res"] = res
    g["small_G"] = frame_state_grads(st, small, res)
    g["small_G_exact"] = frame_state_grads(st, small, res, exact=True)

    # --- (2) planar config-1-shaped slice (16 sensors, 256 balls) ---------
    gx, gy = np.meshgrid(np.arange(4), np.arange(4), indexing="ij")
    ppos = q32(np.column_stack([(gx.ravel() - 1.5) * 2.0,
                                (gy.ravel() - 1.5) * 2.0,
                                np.zeros(16)]))
    planar = SensorArray(ppos, 1.5, 40.0, 2048, 0.0)
    B = 256
    mu = q32(np.column_stack([rng.uniform(-10, 10, B),
                              rng.uniform(-10, 10, B),
                              rng.uniform(10, 30, B)]))
    p0 = q32(rng.uniform(0.1, 1.0, B))
    s_log = 0.3
    a0 = q32(np.clip(rng.lognormal(np.log(0.2) - 0.5 * s_log ** 2, s_log, B),
                     0.1, 0.4))
    mu_obs = q32(mu + rng.normal(0, 0.05, (B, 3)))
    obs = forward_frame(CloudState(a0, p0, mu_obs), planar)
    obs = q32(obs)
    st = CloudState(a0, p0, mu)
    pred = forward_frame(st, planar)
    g["planar_pos"] = ppos
    g["planar_a0"], g["planar_p0"], g["planar_mu"] = a0, p0, mu
    g["planar_obs"] = obs
    g["planar_pred"] = pred
    r = q32(pred - obs)
    g["planar_res"] = r
    g["planar_G"] = frame_state_grads(st, planar, r)

    # --- (3) deformation Jacobians: 3 modes x shared/per-channel ----------
    B, N = 6, 5
    for shared in (True, False):
        theta = q32(rng.uniform(0, 1, (B, N) if shared else (B, 5, N)))
        sigma = q32(rng.uniform(0.05, 0.5, theta.shape))
        omega = q32(rng.uniform(-0.6, 0.6, (B, 5, N)))
        p0 = q32(rng.uniform(0.5, 2.0, B))
        a0 = q32(rng.uniform(0.2, 1.0, B))
        mu = q32(rng.uniform(-4, 4, (B, 3)))
        cloud = DynamicCloud(p0, a0, mu, theta, sigma, omega)
        tag = "sh" if shared else "pc"
        for k, v in (("p0", p0), ("a0", a0), ("mu", mu), ("theta", theta),
                     ("sigma", sigma), ("omega", omega)):
            g[f"def_{tag}_{k}"] = v
        for mode in ("multiplicative", "additive", "radial"):
            s = cloud_states_at(cloud, 0.37, mode, a0_floor=0.3)
            j = cloud_state_grads(cloud, 0.37, mode, a0_floor=0.3)
            key = f"def_{tag}_{mode[:3]}"
            g[key + "_a0t"], g[key + "_p0t"], g[key + "_mut"] = \
                s.a0_t, s.p0_t, s.mu_t
            g[key + "_dbase"] = j.d_base
            g[key + "_domega"] = j.d_omega
            g[key + "_dtheta"] = j.d_theta
            g[key + "_dsigma"] = j.d_sigma
            # chain rule through the radiator on the small array
            resid = q32(rng.normal(0, 1e-3, (8, 64)))
            cg = accumulate_frame_grads(s, j, small, resid)
            g[key + "_res"] = resid
            for nm in ("p0", "a0", "mu", "theta", "sigma", "omega"):
                g[key + "_g" + nm] = getattr(cg, nm)

    # --- (4) Adam: three steps on a fixed gradient sequence ---------------
    p = q32(rng.normal(0, 1, 7))
    grads = q32(rng.normal(0, 1e-2, (3, 7)))
    g["adam_p0"], g["adam_g"] = p.copy(), grads
    st_ = AdamState.like(p)
    traj = []
    for k in range(3):
        adam_step(p, grads[k], st_, lr=1e-2 * (k + 1))
        traj.append(p.copy())
    g["adam_traj"] = np.array(traj)

    # --- (5) prune mask + stable compaction order -------------------------
    pp = q32(rng.uniform(0, 1, 97))
    pp[::7] = q32(pp[::7] * 1e-4)
    g["prune_p0"] = pp
    thr = 1e-2 * float(np.max(pp, initial=0.0))
    keep = pp > thr
    g["prune_keep"] = keep.astype(np.uint8)
    g["prune_order"] = np.nonzero(keep)[0].astype(np.int64)

    # --- (6) three full dynamic iterations (loop + Adam + floors) ---------
    B = 4
    p0 = q32(rng.uniform(0.5, 1.0, B))
    a0 = q32(rng.uniform(0.5, 0.9, B))
    mu = q32(rng.uniform(-4, 4, (B, 3)))
    K = 3
    fr = []
    for k, s in enumerate([1.0, 1.2, 0.9]):
        fr.append(CloudState(a0 * s, p0 * s, mu * s))
    data = np.zeros((8, K, 64))
    for k in range(K):
        data[:, k, :] = forward_frame(fr[k], small)
    data = q32(data)
    obs_set = SignalSet(data, frame_times(K))
    init = [GaussBall(p0[i], a0[i], mu[i]) for i in range(B)]
    cfg = ReconConfig(lr_coords=5e-3, lr_pressure=2e-2, lr_std=2e-3,
                      lr_deform=5e-3, dynamic_iters=3, n_basis=9, seed=2)
    log = []
    cloud = dynamic_reconstruct(obs_set, small, init, cfg,
                                progress=log.append)
    g["dyn_p0"], g["dyn_a0"], g["dyn_mu"] = p0, a0, mu
    g["dyn_data"] = data
    g["dyn_loss"] = np.array([r_["loss"] for r_ in log])
    for nm in ("p0", "a0", "mu", "theta", "sigma", "omega"):
        g["dyn_out_" + nm] = getattr(cloud, nm)

    geometry_and_evaluation(g, q32, small)
    static_stage(g, q32, small)
    file_formats(g)
    ubp_golden(g, q32)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.0f} KiB, {len(g)} arrays)")


def ubp_golden(g, q32):
    """ubp_reconstruct of a simulated frame."""
    from pacloud.core import Box
    from pacloud.deformation import CloudState
    from pacloud.evaluation import GridSpec
    from pacloud.geometry import spherical_array
    from pacloud.radiator import compute_time_window, forward_frame
    from pacloud.reconstruction import ubp_reconstruct
    rng = np.random.default_rng(55)
    roi = Box.cube(4.0)
    arr = spherical_array(48, 25.0, sample_rate=8.0)
    t0, n = compute_time_window(arr, roi, 1.0)
    arr = arr.with_window(t0, n)
    B = 6
    st = CloudState(q32(rng.uniform(0.4, 0.9, B)), q32(rng.uniform(0.3, 1, B)),
                    q32(rng.uniform(-2.5, 2.5, (B, 3))))
    tr = q32(forward_frame(st, arr))
    spec = GridSpec.from_box(roi, 0.5)
    g["ubp_pos"] = arr.positions
    g["ubp_cfg"] = np.array([arr.sound_speed, arr.sample_rate, arr.n_samples,
                             arr.t_start])
    g["ubp_traces"] = tr
    g["ubp_spec"] = np.concatenate([spec.origin, [spec.spacing], spec.dims])
    g["ubp_grid"] = ubp_reconstruct(tr, arr, spec).values


def file_formats(g):
    """PAT1 / GGB1 bytes written by the reference."""
    import tempfile
    from pacloud.core import DynamicCloud, GaussBall
    from pacloud.fileio import write_cloud, write_tensor
    rng = np.random.default_rng(31)
    t = rng.normal(size=(3, 4, 5))
    B, N = 4, 3
    dyn = DynamicCloud(rng.uniform(0.1, 1, B), rng.uniform(0.2, 1, B),
                       rng.normal(size=(B, 3)), rng.uniform(0, 1, (B, N)),
                       rng.uniform(0.1, 0.5, (B, N)),
                       rng.normal(size=(B, 5, N)))
    balls = [GaussBall(0.5, 0.3, [1.0, 2.0, 3.0]),
             GaussBall(0.25, 0.7, [-1.5, 0.0, 0.125])]
    with tempfile.TemporaryDirectory() as d:
        for name, writer, obj in (("pat", write_tensor, t),
                                  ("pat0", write_tensor, np.float64(2.5)),
                                  ("ggb", write_cloud, dyn),
                                  ("ggb_static", write_cloud, balls)):
            p = f"{d}/x"
            writer(p, obj)
            g[f"file_{name}"] = np.frombuffer(open(p, "rb").read(), np.uint8)
    g["file_tensor"] = t
    g["file_dyn_p0"], g["file_dyn_a0"], g["file_dyn_mu"] = dyn.p0, dyn.a0, dyn.mu
    g["file_dyn_theta"], g["file_dyn_sigma"] = dyn.theta, dyn.sigma
    g["file_dyn_omega"] = dyn.omega


def static_stage(g, q32, small):
    """static_reconstruct on the small sphere array
    (lattice init, Adam, floors, one prune that drops balls)."""
    from pacloud.core import Box, ReconConfig
    from pacloud.deformation import CloudState
    from pacloud.radiator import forward_frame
    from pacloud.reconstruction import static_reconstruct
    rng = np.random.default_rng(77)
    B = 3
    st = CloudState(q32(rng.uniform(0.5, 0.9, B)), q32(rng.uniform(0.5, 1, B)),
                    q32(rng.uniform(-2, 2, (B, 3))))
    obs = q32(forward_frame(st, small))
    cfg = ReconConfig(lr_coords=2e-2, lr_pressure=5e-2, lr_std=1e-2,
                      static_iters=6, prune_every=3, prune_threshold=0.9,
                      init_pitch=1.5, init_p0_scale=0.5, step_size=4,
                      drop_rate=0.5, seed=1)
    roi = Box.cube(2.5)
    log = []
    balls = static_reconstruct(obs, small, cfg, roi, progress=log.append)
    g["static_obs"] = obs
    g["static_loss"] = np.array([r["loss"] for r in log])
    g["static_nballs"] = np.array([r["n_balls"] for r in log])
    g["static_p0"] = np.array([b.p0 for b in balls])
    g["static_a0"] = np.array([b.a0 for b in balls])
    g["static_mu"] = np.array([b.mu for b in balls])


def geometry_and_evaluation(g, q32, small):
    """phantoms, arrays, simulate_dataset,
    voxelize, MAP and SSIM from the live reference."""
    from pacloud.core import Box
    from pacloud.deformation import CloudState
    from pacloud.evaluation import (GridSpec, map_project, normalize_pair,
                                    ssim, voxelize)
    from pacloud.geometry import (PhantomSpec, build_phantom,
                                  fibonacci_sphere, simulate_dataset)

    g["geo_fib"] = fibonacci_sphere(37, 12.5)
    specs = {
        "heart": PhantomSpec("heart", Box.cube(12.0), n_frames=3, pitch=1.6,
                             voxel_pitch=1.0),
        "vasc": PhantomSpec("vascular", Box.cube(14.0), n_frames=3,
                            tree_depth=4, seed=3, voxel_pitch=1.0),
        "custom": PhantomSpec("custom", Box.cube(5.0), n_frames=4,
                              pulsation=0.2, voxel_pitch=0.5,
                              custom_balls=((1.0, 0.6, 0.0, 0.0, 0.0),
                                            (0.5, 0.4, 1.5, -1.0, 2.0))),
    }
    for name, spec in specs.items():
        ph = build_phantom(spec)
        g[f"ph_{name}_a0"] = np.stack([f.a0_t for f in ph.frames])
        g[f"ph_{name}_p0"] = np.stack([f.p0_t for f in ph.frames])
        g[f"ph_{name}_mu"] = np.stack([f.mu_t for f in ph.frames])
        g[f"ph_{name}_grid0"] = ph.grids[0].values
        g[f"ph_{name}_gridspec"] = np.concatenate(
            [ph.grids[0].origin, [ph.grids[0].spacing], ph.grids[0].dims])
    # simulate_dataset with noise over the custom phantom (small array)
    ph = build_phantom(specs["custom"])
    sig = simulate_dataset(ph, small, noise_std=1e-3, seed=7)
    g["sim_data"] = sig.data
    # voxelize: a random cloud, fast and exact, odd dims
    rng = np.random.default_rng(99)
    B = 40
    st = CloudState(q32(rng.uniform(0.3, 0.8, B)), q32(rng.uniform(0.2, 1, B)),
                    q32(rng.uniform(-3, 3, (B, 3))))
    spec = GridSpec(np.array([-4.0, -3.5, -4.25]), 0.35, (23, 21, 25))
    g["vox_a0"], g["vox_p0"], g["vox_mu"] = st.a0_t, st.p0_t, st.mu_t
    g["vox_spec"] = np.concatenate([spec.origin, [spec.spacing], spec.dims])
    g["vox_fast"] = voxelize(st, spec).values
    g["vox_exact"] = voxelize(st, spec, exact=True).values
    # MAP + SSIM between the grid and a perturbed copy
    st2 = CloudState(st.a0_t * 1.1, st.p0_t, st.mu_t + 0.2)
    other = voxelize(st2, spec)
    ss = []
    for ax in ("XY", "YZ", "XZ"):
        a, b = normalize_pair(map_project(voxelize(st, spec), ax),
                              map_project(other, ax))
        ss.append(ssim(a, b))
        g[f"map_{ax}"] = map_project(other, ax).values
    g["ssim_vals"] = np.array(ss)


if __name__ == "__main__":
    main()
