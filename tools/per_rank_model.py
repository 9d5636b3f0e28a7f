"""Per-rank compute of frame-sharded runs, measured on ONE GPU (a model of
the N-GPU step, never a multi-GPU measurement): the iteration restricted to
the frames rank 0 would own at N ranks (compute_grads + guarded update +
status read, no collectives), timed with CUDA events.

    python tools/per_rank_model.py [--config 2] [--steps 10]
prints one JSON line: {"config": C, "per_rank_ms": {N: ms}, ...}
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--only", type=int, default=0, help="run only this N")
    args = ap.parse_args()
    from paper_2412_03898_b200 import synth
    from paper_2412_03898_b200.distributed import frame_shard
    from paper_2412_03898_b200.engine import IterationEngine
    from paper_2412_03898_b200.radiator import DeviceArray, forward_device
    dev = torch.device("cuda", 0)
    prob = synth.make_problem(args.config)
    shp = prob.meta["shape"]
    B, M, T, F = shp["B"], shp["M"], shp["T"], shp["F"]
    darr = DeviceArray(prob.array, prob.config.support_sigmas,
                       prob.config.exact_forward)
    obs = torch.empty((F, M, T), dtype=torch.float32, device=dev)
    for k, (a, p, m) in enumerate(prob.gt_frames):
        o, _, _ = forward_device(
            darr, torch.as_tensor(m, device=dev).view(1, B, 3),
            torch.as_tensor(a, dtype=torch.float32, device=dev).view(1, B),
            torch.as_tensor(p, dtype=torch.float32, device=dev).view(1, B))
        obs[k] = o[0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for n in (1, 2, 4, 8):
        if F % n or (args.only and n != args.only):
            continue
        frames = frame_shard(np.arange(F), 0, n)
        eng = IterationEngine(prob.cloud, prob.array, obs, prob.frame_times,
                              prob.config)
        for it in range(3):
            eng.iterate(it, frames)
        torch.cuda.synchronize()
        ts = []
        for it in range(args.steps):
            flush.zero_()
            e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            e0.record()
            eng.iterate(3 + it, frames)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[n] = float(np.mean(ts))
        del eng
        torch.cuda.empty_cache()
    t1 = out.get(1)
    print(json.dumps({"config": args.config, "frames": F, "per_rank_ms": out,
                      "compute_only_efficiency": {n: t1 / (n * t) for n, t in out.items()}
                      if t1 else None}))


if __name__ == "__main__":
    main()
