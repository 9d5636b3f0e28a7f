"""Copy a gpu_job.sh run from gpurun_out/ into profiles/r1/ and regenerate the
measured table in DESIGN.md.  usage: python tools/update_profiles.py TAG"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

tag = sys.argv[1]
out, prof = Path("gpurun_out"), Path("profiles/r1")
for c in (1, 3, 4, 5):
    (prof / f"bench_config{c}.json").write_text(
        (out / f"bench_c{c}.log").read_text().splitlines()[0] + "\n")
(prof / "bench_config2.json").write_text(
    (out / "bench.log").read_text().splitlines()[0] + "\n")
(prof / "bench_config2_reference.json").write_text(
    (out / "bench_ref.log").read_text().splitlines()[0] + "\n")
subprocess.run([sys.executable, "tools/ncu_summary.py", "full",
                str(out / f"prof_{tag}.ncu-rep"),
                str(prof / "ncu_full_config2_fwd_adj.json")], check=True,
               stdout=subprocess.DEVNULL)
subprocess.run([sys.executable, "tools/ncu_summary.py", "launches",
                str(out / "launches.csv"),
                str(prof / "ncu_launches_config2_summary.json")], check=True,
               stdout=subprocess.DEVNULL)
shutil.copy(out / "launches.csv", prof / "ncu_launches_config2.csv")
for suffix, name in (("_all", "ncu_full_config2_all_kernels.json"),
                     ("_c5", "ncu_full_config5_compaction.json")):
    rep = out / f"prof_{tag}{suffix}.ncu-rep"
    if rep.exists():
        subprocess.run([sys.executable, "tools/ncu_summary.py", "full",
                        str(rep), str(prof / name)], check=True,
                       stdout=subprocess.DEVNULL)
full = json.loads((prof / "ncu_full_config2_fwd_adj.json").read_text())
traffic = sum(k["dram_bytes_per_launch"] for k in full)
Path("profiles/ncu_summary.json").write_text(json.dumps({"config2": {
    "dram_bytes_per_launch": traffic,
    "source": "profiles/r1/ncu_full_config2_fwd_adj.json (k_forward + "
              "k_adjoint, one launch each, ncu --set full)"}}, indent=1) + "\n")

rows = {c: json.loads((prof / f"bench_config{c}.json").read_text())
        for c in (1, 2, 3, 4, 5)}
ref = json.loads((prof / "bench_config2_reference.json").read_text())
names = {1: "1 (4k balls, 256 sensors, 1 frame)",
         2: "**2 (20k, 512, 8 frames) — bench default**",
         3: "3 (200k, 1024, 32 frames)",
         4: "4 (1M, 2048, 16 frames, 1 GPU)",
         5: "5 (50k → grows, densify every 8)"}
lines = ["| Config | Iteration (ms) | pair-evals/s | fwd / adj kernel (ms) | "
         "FP32 roofline | e2e (host buffers) | CPU port (cores) |",
         "|---|---|---|---|---|---|---|"]
for c, d in rows.items():
    r, e, cb = d["roofline"], d["e2e"], d.get("cpu_baseline") or {}
    b = "**" if c == 2 else ""
    lines.append(
        f"| {names[c]} | {b}{d['ms_per_step']:.4g}{b} | {b}{d['value']:.3g}{b} | "
        f"{r['t_fwd_ms']:.4g} / {r['t_adj_ms']:.4g} | {b}{100 * r['frac']:.1f} %{b} | "
        f"{e['value']:.3g} /s | {cb.get('value', 0):.2g} /s ({cb.get('cores')})"
        + (f"; reference arm {ref['value']:.2g} /s" if c == 2 else "") + " |")
table = "\n".join(lines) + "\n"
d2 = rows[2]
ratio = (f"Config-2 speed-up of the e2e path over the reference arm (the C "
         f"port of the\nreference's numba kernels on all 16 host cores): "
         f"{d2['e2e']['value']:.3g} / {ref['value']:.3g} ≈ "
         f"{d2['e2e']['value'] / ref['value']:.0f}×.\n")
s = Path("DESIGN.md").read_text()
a = s.index("| Config | Iteration (ms) | pair-evals/s |")
b = s.index("\n\n", a) + 2
s = s[:a] + table + "\n" + s[b:]
a = s.index("Config-2 speed-up of the e2e path")
b = s.index("The e2e leg streams")
s = s[:a] + ratio + s[b:]
Path("DESIGN.md").write_text(s)
print(table + ratio)
