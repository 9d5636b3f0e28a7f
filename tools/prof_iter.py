"""One iteration's dominant launches for ncu (run under ncu with
`--nvtx --nvtx-include "pc_profile/"`): builds BASELINE config C, runs one
untimed engine iteration, then one forward (+ residual + loss) and one
adjoint launch over all frames inside the NVTX range "pc_profile", and, when
WHAT=all, the whole iteration (deform, forward, adjoint, deformation
backward, guard, Adam) eagerly inside the range.

    python tools/prof_iter.py CONFIG [fwdadj|all] [polyfourier|gauss]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2412_03898_b200 import synth  # noqa: E402
from paper_2412_03898_b200.deformation import deform_states_device  # noqa: E402
from paper_2412_03898_b200.engine import IterationEngine  # noqa: E402
from paper_2412_03898_b200.radiator import (DeviceArray, forward_device,  # noqa: E402
                                            state_grads_device)


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    what = sys.argv[2] if len(sys.argv) > 2 else "fwdadj"
    basis = sys.argv[3] if len(sys.argv) > 3 else "polyfourier"
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    prob = synth.make_problem(cfg_id, basis=basis)
    shp = prob.meta["shape"]
    B, M, T, F = shp["B"], shp["M"], shp["T"], shp["F"]
    cfg = prob.config
    darr = DeviceArray(prob.array, cfg.support_sigmas, cfg.exact_forward)
    obs = torch.empty((F, M, T), dtype=torch.float32, device=dev)
    for k, (a, p, m) in enumerate(prob.gt_frames):
        obs[k] = forward_device(
            darr, torch.as_tensor(m, device=dev).view(1, B, 3),
            torch.as_tensor(a, dtype=torch.float32, device=dev).view(1, B),
            torch.as_tensor(p, dtype=torch.float32, device=dev).view(1, B))[0][0]
    del darr
    eng = IterationEngine(prob.cloud, prob.array, obs, prob.frame_times, cfg,
                          use_graph=False, spatial_order=cfg_id != 5)
    frames = np.arange(F)
    eng.iterate(0, frames)
    torch.cuda.synchronize()
    nvtx = torch.cuda.nvtx
    if what == "all":
        nvtx.range_push("pc_profile")
        eng.iterate(1, frames)
        nvtx.range_pop()
    else:
        eng._ensure_buffers(F)
        eng.t_dev.copy_(torch.as_tensor(prob.frame_times))
        deform_states_device(eng.dcloud, eng.t_dev, cfg.coord_mode,
                             cfg.a0_floor, eng.mu_t, eng.a0_t, eng.p0_t, eng.H)
        torch.cuda.synchronize()
        nvtx.range_push("pc_profile")
        forward_device(eng.darr, eng.mu_t, eng.a0_t, eng.p0_t,
                       observed=eng.observed, out=eng.resid, loss=eng.loss_f,
                       coincident=eng.coinc, workspace=eng.ws)
        state_grads_device(eng.darr, eng.mu_t, eng.a0_t, eng.p0_t, eng.resid,
                           G=eng.G, coincident=eng.coinc)
        nvtx.range_pop()
    torch.cuda.synchronize()
    print("profiled config", cfg_id, what)


if __name__ == "__main__":
    main()
