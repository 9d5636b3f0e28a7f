"""The TMA-staged register-run forward (PC_FWD_TMA=1: fwd_run.cu compiled with
PC_FR_TMA, the chunk's raw ball tile copied into shared memory by
cp.async.bulk behind an mbarrier while the previous chunk's runs are swept)
against the oracle and against the default forward.

The variant is chosen once per process, so each case runs in a child
process.  Cases: ball counts that are whole 16-byte multiples (every chunk
staged), an odd ball count (odd frames misaligned -> plain-load fallback for
those frames, staged for the even ones), a tail chunk of < 4 balls, exact
mode (direct path).  radiator.py:86-118 is the loop being replaced."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import oracle
from paper_2412_03898_b200 import synth
from paper_2412_03898_b200.radiator import DeviceArray, forward_device
out = {}
dev = torch.device("cuda", 0)
for name, B, F, exact in (("aligned", 1536, 3, False), ("odd", 1501, 4, False),
                          ("tail", 1026, 2, False), ("exact", 600, 2, True)):
    prob = synth.make_problem(2, seed=31, n_balls=B, n_sensors=24, n_frames=F,
                              n_samples=4096)
    cfg = prob.config
    darr = DeviceArray(prob.array, cfg.support_sigmas, exact)
    variant = darr.variant()
    a = np.stack([f[0] for f in prob.gt_frames]); p = np.stack([f[1] for f in prob.gt_frames])
    m = np.stack([f[2] for f in prob.gt_frames])
    got = forward_device(darr, torch.as_tensor(m, device=dev),
                         torch.as_tensor(a, dtype=torch.float32, device=dev),
                         torch.as_tensor(p, dtype=torch.float32, device=dev))[0].cpu().numpy()
    ref = np.stack([oracle.forward_frame(
        oracle.States(a[k].astype(np.float32).astype(np.float64),
                      p[k].astype(np.float32).astype(np.float64), m[k]),
        prob.array, exact=exact) for k in range(F)])
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    np.save(sys.argv[2] + "_" + name + ".npy", got)
    out[name] = {"rel": rel, "variant": variant}
print("RESULT " + json.dumps(out))
"""


def _run(tmp_path, tag, tma):
    env = dict(os.environ)
    env.pop("PC_FWD_LEGACY", None)
    if tma:
        env["PC_FWD_TMA"] = "1"
    else:
        env.pop("PC_FWD_TMA", None)
    script = tmp_path / "child.py"
    script.write_text(CHILD)
    r = subprocess.run([sys.executable, str(script), str(ROOT), str(tmp_path / tag)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    return json.loads(line[7:])


def test_tma_staged_forward_matches_oracle_and_default(tmp_path):
    import numpy as np
    tma = _run(tmp_path, "tma", True)
    base = _run(tmp_path, "base", False)
    for name in ("aligned", "odd", "tail", "exact"):
        assert tma[name]["variant"] == 2, tma[name]     # the staged kernel ran
        assert base[name]["variant"] == 0
        assert tma[name]["rel"] < 1e-5, (name, tma[name])
        assert base[name]["rel"] < 1e-5, (name, base[name])
        a = np.load(str(tmp_path / f"tma_{name}.npy"))
        b = np.load(str(tmp_path / f"base_{name}.npy"))
        # the two differ only in the chunk size (512 vs 1024 balls per
        # partial sum): fp32 summation order
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 2e-6, name
