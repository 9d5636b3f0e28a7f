"""bench.py contract: the reference arm (the CPU port of the reference
algorithm) prints one well-formed JSON line without a GPU; the measured arm
(GPU) prints one line with every key the contract asks for."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
         "--config", "1", "--steps", "1", "--warmup", "1",
         "--cpu-sensors", "8"],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
                "ms_per_step", "higher_is_better", "scaling", "dtype",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["value"] > 0
    assert line["config"]["workload"] == "BASELINE config 1"


@pytest.mark.gpu
def test_ours_json_line_on_gpu():
    """The measured arm on config 1: one JSON line with every key the
    contract asks for (roofline with traffic and pipe ceiling, cpu_baseline,
    e2e with byte counts, gpu_launches, clocks)."""
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--config", "1",
         "--steps", "3", "--warmup", "3", "--cpu-sensors", "8"],
        capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
                "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
                "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in line, key
    r = line["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic",
                "pipe_ceiling"):
        assert key in r, key
    assert 0 < r["frac"] < 1 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["cpu_baseline"]["cores"] >= 1
