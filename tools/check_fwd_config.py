"""Full-size forward parity of one frame against the CPU oracle (GPU box).

usage: python tools/check_fwd_config.py CONFIG [n_sensors_subsample]
Prints rel-L2 and max |err| / peak of the predicted traces for frame 0."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2412_03898_b200 import synth  # noqa: E402
from paper_2412_03898_b200.core import SensorArray  # noqa: E402
from paper_2412_03898_b200.radiator import DeviceArray, forward_device  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
every = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prob = synth.make_problem(cfg, seed=cfg)
a0, p0, mu = prob.gt_frames[0]
arr = prob.array
sub = SensorArray(arr.positions[::every], arr.sound_speed, arr.sample_rate,
                  arr.n_samples, arr.t_start)
dev = torch.device("cuda")
darr = DeviceArray(sub, 6.0, False)
mu_t = torch.as_tensor(mu, device=dev)[None].contiguous()
a0_t = torch.as_tensor(a0, dtype=torch.float32, device=dev)[None].contiguous()
p0_t = torch.as_tensor(p0, dtype=torch.float32, device=dev)[None].contiguous()
out, _, _ = forward_device(darr, mu_t, a0_t, p0_t)
got = out[0].double().cpu().numpy()
t = time.time()
ref = oracle.forward_frame(oracle.States(a0.astype(np.float32).astype(np.float64),
                                         p0.astype(np.float32).astype(np.float64), mu), sub)
err = got - ref
print(f"config {cfg}: B={len(p0)} M={sub.n_sensors} T={sub.n_samples} "
      f"rel_l2={np.linalg.norm(err) / np.linalg.norm(ref):.3e} "
      f"max_err/peak={np.abs(err).max() / np.abs(ref).max():.3e} "
      f"oracle {time.time() - t:.1f}s")
