"""Full (not extrapolated) CPU reference iteration, BASELINE.md step 3 for
configs 1-2: every frame, every sensor, every ball through the reference
algorithm's CPU port (oracle/: deformation + forward + residual + adjoint +
chain rule, fp64, all host threads).  Min of `reps` iterations.

    python tools/ref_full.py CONFIG [REPS]  -> one JSON line
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2412_03898_b200 import synth  # noqa: E402


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    prob = synth.make_problem(cfg_id)
    threads = os.cpu_count() or 1
    arr = prob.array
    obs = np.stack([oracle.forward_frame(oracle.States(a, p, m), arr,
                                         threads=threads)
                    for a, p, m in prob.gt_frames])
    shp = prob.meta["shape"]
    times, loss = [], None
    for _ in range(reps):
        t = time.perf_counter()
        loss, _ = oracle.iteration_grads(prob.cloud, prob.frame_times, obs,
                                         arr, prob.config,
                                         basis=prob.cloud.basis)
        times.append(time.perf_counter() - t)
    best = min(times)
    pairs = shp["B"] * shp["M"] * shp["F"]
    print(json.dumps({
        "impl": "reference", "kind": "port", "config": cfg_id,
        "what": "full iteration (all frames, sensors, balls): deform + "
                "forward + residual/loss + adjoint + chain rule, fp64",
        "cores": threads, "reps": reps, "iteration_s": times,
        "iteration_s_min": best, "pair_evals_per_s": pairs / best,
        "loss": float(loss), "extrapolated": False}))


if __name__ == "__main__":
    main()
