"""Benchmark: BASELINE metric "ball x sensor pair-evals/s (fwd+adjoint) and
iteration ms" on BASELINE config 3 (default: the largest single-GPU config and
the BASELINE's frame-sharded 1/2/4/8-GPU case; `--config` selects others).

One step = one full 4D iteration through the fused engine: deform ->
forward + residual + L2 loss -> adjoint -> deformation backward ->
[NCCL all-reduce] -> finite guard + the iteration's single host sync ->
Adam/floors.  value = B*M*F pair-evals of the whole job per second of step
time (max over ranks).  Inputs are seeded synthetic scenes
(paper_2412_03898_b200.synth); L2 is flushed (a 256 MiB write) between timed
steps, outside each step's CUDA-event bracket.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C]
    python bench.py --impl reference ...   # CPU oracle port, host threads
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ball x sensor pair-evals/s (fwd+adjoint), full 4D iteration"
UNIT = "pair-evals/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
NCU_SUMMARY = ROOT / "profiles" / "ncu_summary.json"
FLOPS_PER_SAMPLE = 20.0     # fwd 7 + adj 13 canonical flops


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sensors", type=int, default=0)
    ap.add_argument("--densify-every", type=int, default=8,
                    help="config 5: densify/prune every N iterations")
    ap.add_argument("--max-balls", type=int, default=500000,
                    help="config 5: growth cap")
    ap.add_argument("--basis", default="polyfourier",
                    choices=["polyfourier", "gauss"],
                    help="deformation basis: BASELINE's poly+Fourier (N=8) "
                         "or the reference default Gaussian basis")
    ap.add_argument("--n-basis", type=int, default=None,
                    help="Gaussian basis size (reference default 65)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def sm_peak_fp32():
    """FP32 FMA peak: 148 SMs x 128 lanes x 2 flop x max SM clock."""
    mhz = 1965.0
    src = "derived: 148 SM x 128 FP32 lanes x 2 flop x 1965 MHz (sm_max_mhz)"
    if PEAKS.exists():
        try:
            mhz = float(json.loads(PEAKS.read_text()).get("sm_max_mhz", mhz))
            src = (f"derived: 148 SM x 128 FP32 lanes x 2 flop x {mhz:.0f} MHz"
                   f" (MEASURED_PEAKS.json sm_max_mhz)")
        except Exception:
            pass
    return 148 * 128 * 2 * mhz * 1e6 / 1e12, src


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,"
         "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/pacloud_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=self.fh, stderr=subprocess.DEVNULL)
            # sampler up (first line written) before the timed region starts
            t_end = time.time() + 3.0
            while time.time() < t_end and self.proc.poll() is None and \
                    self.path.stat().st_size == 0:
                time.sleep(0.01)
            self.skip = self.path.read_text().count("\n")
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None and \
                self.path.read_text().count("\n") <= getattr(self, "skip", 0):
            # timed region shorter than the sampling interval: one sample
            # taken synchronously as it ends
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True,
                    text=True, timeout=10).stdout
                self.extra = out.strip().splitlines()
            except Exception:
                self.extra = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        lines = self.path.read_text().splitlines()[getattr(self, "skip", 0):]
        for line in lines + list(getattr(self, "extra", [])):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def support_samples_torch(mu_t, a0_t, pos, v, t0, dt, T, support=6.0):
    """Exact in-support sample count (radiator.py:103-110) on the device,
    as measurement plumbing (torch), frame by frame."""
    import torch
    total = 0
    for f in range(mu_t.shape[0]):
        for b0 in range(0, mu_t.shape[1], 65536):
            mu = mu_t[f, b0:b0 + 65536]
            a0 = a0_t[f, b0:b0 + 65536].double()
            R = torch.cdist(mu, pos)                       # (b, M) f64
            sa = support * a0[:, None]
            lo = torch.ceil(((R - sa) / v - t0) / dt).clamp(0, T)
            hi = (torch.floor(((R + sa) / v - t0) / dt) + 1).clamp(0, T)
            total += int((hi - lo).clamp_min(0).sum().item())
    return total


def full_support_initial(prob, dev):
    """Sum over every (ball, sensor, frame) of the in-support window length
    for the problem's initial cloud (the states the CPU sample is drawn
    from), counted on the device (measurement plumbing; states from the
    oracle's deformation restatement)."""
    import oracle
    import torch
    cfg = prob.config
    pos = torch.as_tensor(prob.array.positions, dtype=torch.float64,
                          device=dev)
    dt = 1.0 / prob.array.sample_rate
    total = 0
    for t in prob.frame_times:
        st = oracle.cloud_states_at(prob.cloud, float(t), cfg.coord_mode,
                                    cfg.a0_floor, basis=prob.cloud.basis)
        total += support_samples_torch(
            torch.as_tensor(st.mu_t, device=dev)[None],
            torch.as_tensor(st.a0_t, device=dev)[None], pos,
            prob.array.sound_speed, prob.array.t_start, dt,
            prob.array.n_samples, cfg.support_sigmas)
    return total


class CpuSample:
    """The reference algorithm's CPU port (oracle/, the C restatement of the
    numba kernels radiator.py:86-174) on a bounded, deterministic sample of
    one iteration: frame 0 (deformed states), every k-th sensor, all balls,
    forward + adjoint in fp64 on `threads` host threads.  The full
    iteration's time is extrapolated by in-support samples (SURVEY.md 8d:
    the port's cost is linear in the window samples), so `value` is the
    pair-evals/s the port would reach on the whole iteration."""

    def __init__(self, prob, n_sensors, threads, full_support=None):
        import oracle
        from paper_2412_03898_b200.core import SensorArray
        cfg = prob.config
        self.threads = threads
        self.st = oracle.cloud_states_at(prob.cloud, float(prob.frame_times[0]),
                                         cfg.coord_mode, cfg.a0_floor,
                                         basis=prob.cloud.basis)
        M = prob.array.n_sensors
        step = max(1, M // max(1, n_sensors))
        sel = np.arange(0, M, step)[:n_sensors]
        self.sub = SensorArray(prob.array.positions[sel],
                               prob.array.sound_speed, prob.array.sample_rate,
                               prob.array.n_samples, prob.array.t_start)
        a, p, m = prob.gt_frames[0]
        self.obs = oracle.forward_frame(oracle.States(a, p, m), self.sub,
                                        threads=threads)
        self.s_sample = oracle.support_samples(self.st, self.sub,
                                               cfg.support_sigmas,
                                               threads=threads)
        shp = prob.meta["shape"]
        self.pairs_full = shp["B"] * shp["M"] * shp["F"]
        if full_support is None:
            full_support = 0
            for k in range(shp["F"]):
                stk = oracle.cloud_states_at(
                    prob.cloud, float(prob.frame_times[k]), cfg.coord_mode,
                    cfg.a0_floor, basis=prob.cloud.basis)
                full_support += oracle.support_samples(
                    stk, prob.array, cfg.support_sigmas, threads=threads)
        self.s_full = int(full_support)
        self.desc = (f"frame 0, {len(sel)} of {M} sensors (every {step}th), "
                     f"all {len(self.st.a0_t)} balls: oracle fwd+adjoint "
                     f"fp64 on {threads} threads; extrapolated to the full "
                     f"iteration by in-support samples "
                     f"({self.s_full:.4e} / {self.s_sample:.4e})")

    def time_once(self):
        import oracle
        t = time.perf_counter()
        pred = oracle.forward_frame(self.st, self.sub, threads=self.threads)
        oracle.frame_state_grads(self.st, self.sub, pred - self.obs,
                                 threads=self.threads)
        return time.perf_counter() - t

    def value(self, secs):
        """pair-evals/s of the whole iteration extrapolated from `secs`."""
        return self.pairs_full / (secs * self.s_full / self.s_sample)


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU port (the reference
    is pure Python/numba; its C restatement in oracle/ is timed), each step
    one bounded sample of the iteration, extrapolated by in-support
    samples."""
    if rank != 0:
        return
    from paper_2412_03898_b200 import synth
    prob = synth.make_problem(args.config, seed=args.seed, basis=args.basis,
                              n_basis=args.n_basis)
    threads = os.cpu_count() or 1
    # ~1.3 s of 16-thread work per step at config 3 (13 steps: ~17 s)
    n_s = args.cpu_sensors or {3: 32, 4: 8, 5: 32}.get(args.config, 128)
    samp = CpuSample(prob, n_s, threads)
    for _ in range(max(1, args.warmup)):
        samp.time_once()
    t0 = time.perf_counter()
    secs = [samp.time_once() for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    value = samp.value(float(np.median(secs)))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * samp.pairs_full / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, fp32-quantised)",
        "config": workload_config(args.config, prob, world),
        "extrapolated": True,
        "cpu_baseline": {"value": value, "unit": UNIT,
                         "cores": threads, "kind": "port",
                         "sample": samp.desc, "extrapolated": True,
                         "sample_s_median": float(np.median(secs))},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg_id, prob, world):
    shp = prob.meta["shape"]
    shard = "sensors" if (cfg_id == 4 or shp["F"] < world) else "frames"
    return {"workload": f"BASELINE config {cfg_id}",
            "balls": shp["B"], "sensors": shp["M"], "samples": shp["T"],
            "frames": shp["F"], "basis": prob.cloud.basis,
            "n_basis": int(prob.cloud.n_basis),
            "coord_mode": prob.config.coord_mode,
            "parallelism": f"{shard}-sharded x{world}" if world > 1
            else "single GPU",
            "l2": "flushed (256 MiB write) between timed steps"}


def run_ours(args, rank, world, local):
    import torch
    from paper_2412_03898_b200 import _lib, synth
    from paper_2412_03898_b200.distributed import frame_shard, shard_range
    from paper_2412_03898_b200.engine import IterationEngine
    from paper_2412_03898_b200.radiator import DeviceArray, forward_device

    # one process per GPU; PC_DIST_BACKEND=gloo with more ranks than GPUs is
    # a functional check of the sharded path only (never a measurement)
    backend = os.environ.get("PC_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" \
        else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime
        kw = {"device_id": dev} if backend == "nccl" else {}
        torch.distributed.init_process_group(
            backend, timeout=datetime.timedelta(minutes=10), **kw)
    prob = synth.make_problem(args.config, seed=args.seed, basis=args.basis,
                              n_basis=args.n_basis)
    shp = prob.meta["shape"]
    B, M, T, F = shp["B"], shp["M"], shp["T"], shp["F"]
    arr = prob.array
    cfg = prob.config

    # ---- observed traces: forward-simulate the ground-truth frames on the
    # device (input synthesis, not timed; simulate_dataset geometry.py:266)
    darr_full = DeviceArray(arr, cfg.support_sigmas, cfg.exact_forward)
    obs = torch.empty((F, M, T), dtype=torch.float32, device=dev)
    for k, (a, p, m) in enumerate(prob.gt_frames):
        o, _, _ = forward_device(
            darr_full, torch.as_tensor(m, device=dev).view(1, B, 3),
            torch.as_tensor(a, dtype=torch.float32, device=dev).view(1, B),
            torch.as_tensor(p, dtype=torch.float32, device=dev).view(1, B))
        obs[k] = o[0]
    del darr_full

    # sensors are sharded for config 4 and whenever the frames cannot cover
    # the ranks (config 1 has one frame)
    sensor_shard = world > 1 and (args.config == 4 or F < world)
    frames_all = np.arange(F)
    if sensor_shard:
        lo, hi = shard_range(M, rank, world)
        eng = IterationEngine(prob.cloud, arr, obs[:, lo:hi].contiguous(),
                              prob.frame_times, cfg, shard="sensors")
        local_frames = frames_all
    else:
        local_frames = frame_shard(frames_all, rank, world)
        eng = IterationEngine(prob.cloud, arr, obs, prob.frame_times, cfg,
                              shard="frames",
                              spatial_order=args.config != 5)
    del obs
    torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    it = 0

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    growth = []

    def step(it):
        """One iteration (+ the config-5 densify/prune when due)."""
        eng.iterate(it, frames_all)
        if args.config == 5 and (it + 1) % args.densify_every == 0:
            eng.densify(p0_min=0.01, q=90.0, max_balls=args.max_balls)
            growth.append((it, eng.B))

    for _ in range(args.warmup):
        step(it)
        it += 1
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step CUDA events, L2 flushed between
    ev = [(torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    pairs_done = 0
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            flush.zero_()
            pairs_done += eng.B * M * F
            ev[k][0].record()
            step(it)
            ev[k][1].record()
            it += 1
        torch.cuda.synchronize()
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if os.environ.get("PC_BENCH_DEBUG"):
        print("step ms", [round(x, 3) for x in step_ms], "B", eng.B,
              "mem MB", torch.cuda.memory_allocated() >> 20,
              "peak MB", torch.cuda.max_memory_allocated() >> 20, file=sys.stderr)
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    pairs = pairs_done / args.steps            # per step (B grows in config 5)
    value = pairs / (ms * 1e-3)

    # ---- dominant kernels: fwd + adj, timed live with events on the
    # launching stream (eager, same buffers), and exact algorithmic work
    F_loc = len(local_frames)
    eng._ensure_buffers(F_loc)          # B may have changed (config-5 densify)
    eng.t_dev.copy_(torch.as_tensor(prob.frame_times[local_frames]))
    from paper_2412_03898_b200.deformation import deform_states_device
    from paper_2412_03898_b200.radiator import state_grads_device
    deform_states_device(eng.dcloud, eng.t_dev, cfg.coord_mode, cfg.a0_floor,
                         eng.mu_t, eng.a0_t, eng.p0_t, eng.H)
    obs_loc = eng.observed[int(local_frames[0]):int(local_frames[0]) + F_loc] \
        if not sensor_shard else eng.observed
    reps = 5
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_fwd = t_adj = 0.0
    for r in range(reps + 1):
        flush.zero_()
        e[0].record()
        forward_device(eng.darr, eng.mu_t, eng.a0_t, eng.p0_t, observed=obs_loc,
                       out=eng.resid, loss=eng.loss_f, coincident=eng.coinc,
                       workspace=eng.ws)
        e[1].record()
        state_grads_device(eng.darr, eng.mu_t, eng.a0_t, eng.p0_t, eng.resid,
                           G=eng.G, coincident=eng.coinc)
        e[2].record()
        torch.cuda.synchronize()
        if r:
            t_fwd += e[0].elapsed_time(e[1]) / reps
            t_adj += e[1].elapsed_time(e[2]) / reps
    B = eng.B
    S = support_samples_torch(eng.mu_t, eng.a0_t, eng.darr.positions,
                              eng.darr.v, eng.darr.t0, eng.darr.dt,
                              eng.darr.T, cfg.support_sigmas)
    peak, peak_src = sm_peak_fp32()
    achieved = FLOPS_PER_SAMPLE * S / ((t_fwd + t_adj) * 1e-3) / 1e12
    traffic = None
    if NCU_SUMMARY.exists():
        try:
            summ = json.loads(NCU_SUMMARY.read_text())
            traffic = summ.get(f"config{args.config}", {}).get(
                "dram_bytes_per_launch")
        except Exception:
            traffic = None
    kern_pairs = B * eng.darr.M * F_loc
    roofline = {
        "bound": "fp32", "unit": "TFLOP/s", "achieved": achieved,
        "peak": peak, "frac": achieved / peak, "traffic": traffic,
        "kernel": "k_fwd_run + k_adjoint (every forward and adjoint launch of one iteration on the local shard)",
        "flops_per_launch": FLOPS_PER_SAMPLE * S,
        "support_samples": S, "t_fwd_ms": t_fwd, "t_adj_ms": t_adj,
        "kernel_pair_evals_per_s": kern_pairs / ((t_fwd + t_adj) * 1e-3),
        "mufu_frac": 2.0 * S / ((t_fwd + t_adj) * 1e-3) /
        (148 * 16 * 1965e6),
        "peak_source": peak_src,
        # the algorithm's pipe ceiling: forward bound by
        # the shared-memory float2 read-modify-write and adjoint by the
        # FMA/MUFU balance, both measured at ~16 in-support samples / clk /
        # SM (tools/ubench/pipes.cu, profiles/r1/ubench_pipes_b200.txt)
        "pipe_ceiling": {
            "frac": FLOPS_PER_SAMPLE * 8.0 / 256.0,
            "frac_achieved_of_ceiling": (achieved / peak) / (FLOPS_PER_SAMPLE * 8.0 / 256.0),
            "samples_per_clk_per_sm": S / ((t_fwd + t_adj) * 1e-3) / (148 * 1965e6),
            "ceiling_samples_per_clk_per_sm": 8.0,
        },
    }

    # ---- e2e: the user-facing call with host buffers (pinned observed in,
    # loss out), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        # observed traces live in pinned host memory; every step uploads the
        # frames it uses (side stream, overlapped with deform + forward sweep)
        host_obs = eng.observed.cpu().pin_memory()
        eng.stream_observed_from(host_obs)
        n_loc = len(eng._local_frames(frames_all))
        h2d = n_loc * host_obs[0].numel() * host_obs.element_size()
        for _ in range(args.warmup):         # re-capture with the upload
            eng.iterate(it, frames_all)
            it += 1
        barrier()
        torch.cuda.synchronize()
        ee = [(torch.cuda.Event(enable_timing=True),
               torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        losses = []
        e2e_pairs = 0
        for k in range(args.steps):
            flush.zero_()
            e2e_pairs += eng.B * M * F
            ee[k][0].record()
            losses.append(eng.iterate(it, frames_all))   # H2D obs, D2H loss
            if args.config == 5 and (it + 1) % args.densify_every == 0:
                eng.densify(p0_min=0.01, q=90.0, max_balls=args.max_balls)
            ee[k][1].record()
            it += 1
        torch.cuda.synchronize()
        e2e_step_ms = [a.elapsed_time(b) for a, b in ee]
        if os.environ.get("PC_BENCH_DEBUG"):
            print("e2e step ms", [round(x, 3) for x in e2e_step_ms], "B", eng.B,
                  file=sys.stderr)
        ems = float(np.mean(e2e_step_ms))
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": e2e_pairs / args.steps / (ems * 1e-3), "unit": UNIT,
               "ms_per_step": ems,
               "h2d_bytes_per_step": int(h2d) + eng._hyper_host.numel() * eng._hyper_host.element_size(),
               "d2h_bytes_per_step": eng._status_host.numel() * eng._status_host.element_size(),
               "api": "IterationEngine.iterate with the step's observed frames "
                      "uploaded from pinned host memory (stream_observed_from)"}
        eng.stream_observed_from(None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        # ~5 s of 16-thread work per pass at config 3 (3 passes: ~15 s)
        n_s = args.cpu_sensors or {3: 128, 4: 32, 5: 128}.get(args.config, 512)
        samp = CpuSample(prob, n_s, threads,
                         full_support=full_support_initial(prob, dev))
        samp.time_once()
        secs = min(samp.time_once() for _ in range(2))
        cpu = {"value": samp.value(secs), "unit": UNIT, "cores": threads,
               "kind": "port", "sample": samp.desc + ", min of 2",
               "extrapolated": True}

    # deform + forward[+combine]+loss-reduce + adjoint + deform-bwd + finite
    # guard + Adam
    launches_per_step = 5 + eng.darr.plan(B, F_loc)["launches"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded, fp32-quantised; observed traces "
                    "forward-simulated from ground-truth frames)",
            "config": workload_config(args.config, prob, world),
            "iteration_ms": ms, "step_ms_min": float(np.min(step_ms)),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "final_loss": float(eng.loss_total.item()),
            "final_balls": int(eng.B),
        }
        if args.config == 5:
            # per-step times: densify steps (prune/split + gathers; the next
            # step re-captures the graphs at the new ball count) vs the rest
            first = args.warmup
            dens = {i - first for i, _ in growth if i >= first}
            after = {i + 1 for i in dens}
            plain = [t for i, t in enumerate(step_ms)
                     if i not in dens and i not in after]
            line["growth"] = {
                "densify_every": args.densify_every,
                "balls_at_densify": [b for _, b in growth],
                "step_ms_plain_mean": float(np.mean(plain)) if plain else None,
                "step_ms_densify_mean": float(np.mean(
                    [step_ms[i] for i in dens])) if dens else None,
                "step_ms_after_densify_mean": float(np.mean(
                    [step_ms[i] for i in after if i < len(step_ms)]))
                if after else None,
                "step_ms": [round(t, 3) for t in step_ms]
                if len(step_ms) <= 400 else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
