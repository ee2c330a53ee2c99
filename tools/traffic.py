"""Per-kernel DRAM traffic and duration of one bench step, from an ncu metric pass
(cold-cache, serialised launches; not a bench number). Writes profiles/r02_traffic_<wl>.json,
which bench.py cites in its roofline object (traffic of the dominant kernel, and for the
traceback kernels the readback bytes over their time).

python tools/traffic.py <workload> [--steps 1]     (runs ncu itself; GPU box only)
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def main(wl: str, parse_only: bool = False):
    """Run the ncu metric pass (GPU box) unless parse_only, then summarise the CSV
    gpurun_out/traffic_<wl>.csv into profiles/r02_traffic_<wl>.json."""
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{wl}.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    if not parse_only:
        cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "--csv", "--log-file", log,
               sys.executable, "bench.py", "--workload", wl, "--steps", "1", "--warmup", "3",
               "--no-cpu", "--no-check"]
        subprocess.run(cmd, cwd=ROOT, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO("".join(l for l in open(log) if l.startswith('"')))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(lambda: defaultdict(list))  # kernel -> metric -> values (one per launch)
    order = []
    for r in rows[1:]:
        name = r[ix["Kernel Name"]]
        if "nwk::" not in name and "k_" not in name:
            continue
        short = name.split("(")[0].replace("void ", "").replace("nwk::", "")
        if short not in per:
            order.append(short)
        val = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
                 "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        per[short][r[ix["Metric Name"]]].append(val * scale)
    # the last launches are the timed step (warm-up steps come first): keep per-launch means
    out = {"workload": wl, "source": "ncu --metrics " + METRICS + " (cold cache, serialised)",
           "kernels": {}}
    for k in order:
        m = per[k]
        n = len(m["gpu__time_duration.sum"])
        rd = sum(m["dram__bytes_read.sum"]) / n
        wr = sum(m["dram__bytes_write.sum"]) / n
        ns = sum(m["gpu__time_duration.sum"]) / n
        out["kernels"][k] = {"launches_captured": n, "dram_read_bytes_per_launch": rd,
                             "dram_write_bytes_per_launch": wr, "ns_per_launch": ns,
                             "GBps": (rd + wr) / ns if ns else None}
    dst = os.path.join(ROOT, "profiles", f"r02_traffic_{wl}.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[-1], parse_only="--parse" in sys.argv)
