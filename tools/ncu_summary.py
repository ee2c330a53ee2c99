"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into a small text file
for profiles/ (the numbers bench.py's roofline cites).

python tools/ncu_summary.py report.ncu-rep > profiles/rNN_<name>.txt
python tools/ncu_summary.py --launches launches.csv > profiles/rNN_launches.txt
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
]
STALLS = ["smsp__pcsamp_warps_issue_stalled_" + s for s in (
    "selected", "wait", "long_scoreboard", "short_scoreboard", "no_instructions",
    "branch_resolving", "sleeping", "membar", "math_pipe_throttle", "dispatch_stall", "mio_throttle")]


def report(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append(f"kernel: {d.get('Kernel Name', '?')[:110]}")
        for m in METRICS:
            if m in d:
                out.append(f"  {m:62s} {d[m]:>20s} {u.get(m, '')}")
        tot = sum(float(d.get(s, 0) or 0) for s in STALLS)
        if tot:
            out.append("  warp-state samples (share):")
            for s in STALLS:
                v = float(d.get(s, 0) or 0)
                if v:
                    out.append(f"    {s.split('stalled_')[1]:24s} {100 * v / tot:6.1f}%")
    return "\n".join(out)


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0.0, 0])
    unit = ""
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"][:80]
                agg[k][0] += float(d["Metric Value"].replace(",", ""))
                agg[k][1] += 1
                unit = d.get("Metric Unit", "")
    tot = sum(v[0] for v in agg.values()) or 1.0
    out = [f"# launch list (ncu --metrics gpu__time_duration.sum, cold-cache serialised), unit {unit}",
           f"# {'avg/launch':>14s} {'launches':>8s} {'share':>7s}  kernel"]
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        out.append(f"  {v / n:14.1f} {n:8d} {100 * v / tot:6.1f}%  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[1]))
