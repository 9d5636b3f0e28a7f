"""Summarise ncu captures for profiles/ (run in the build container).

    python tools/ncu_summary.py full  <report.ncu-rep | raw.csv> <out.json>
    python tools/ncu_summary.py launches <launches.csv> <out.json>

`full`: per kernel the time, pipe utilisations, issue efficiency, DRAM
bytes (read + write = the roofline `traffic`), occupancy and the top stall
reasons.  `launches`: the `--metrics gpu__time_duration.sum` launch list
grouped by kernel, with each kernel's share of the captured time.
"""

import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "time_ms": "gpu__time_duration.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_mufu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "registers": "launch__registers_per_thread",
    "sm_mhz": "smsp__cycles_elapsed.avg.per_second",
}
def _hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json), else the recipe's
    fallback."""
    try:
        return float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
    except Exception:
        return 6531.9


HBM_GBS = _hbm_peak()
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0,
         "us": 1e-3, "ms": 1.0, "ns": 1e-6, "s": 1e3}


def full(rep, out):
    if rep.endswith(".csv"):          # `ncu -i X --page raw --csv` exported on the box
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                             capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d["Kernel Name"]}
        for name, key in KEYS.items():
            if key not in d:
                continue
            try:
                v = float(d[key].replace(",", ""))
            except ValueError:
                continue
            if name.startswith("dram"):
                v *= SCALE.get(u[key], 1.0)
            if name == "time_ms":
                v *= SCALE.get(u[key], 1.0)
            k[name] = v
        if "dram_read" in k:
            k["dram_bytes_per_launch"] = k["dram_read"] + k.get("dram_write", 0)
            if k.get("time_ms"):
                gbs = k["dram_bytes_per_launch"] / (k["time_ms"] * 1e-3) / 1e9
                k["dram_gbps"] = round(gbs, 1)
                k["hbm_frac"] = round(gbs / HBM_GBS, 4)
        stalls = []
        for key, v in d.items():
            if key.startswith("smsp__pcsamp_warps_issue_stalled") and \
                    not key.endswith("not_issued"):
                try:
                    stalls.append((float(v), key.split("stalled_")[-1]))
                except ValueError:
                    pass
        tot = sum(x for x, _ in stalls) or 1.0
        k["top_stalls_pct"] = {n: round(100 * x / tot, 1)
                               for x, n in sorted(stalls, reverse=True)[:6]}
        res.append(k)
    json.dump(res, open(out, "w"), indent=1)
    return res


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Value"),
                  hdr.index("Metric Unit"))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * {"nsecond": 1e-6, "usecond": 1e-3,
                                             "msecond": 1.0}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values()) or 1.0
    res = {n: {"launches": c, "total_ms": t, "share": t / tot}
           for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    json.dump(res, open(out, "w"), indent=1)
    return res


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    print(json.dumps((full if mode == "full" else launches)(src, dst),
                     indent=1)[:2000])
