"""Summarise ncu --set full captures (one kernel launch each) into profiles/ncu_summary.json (tracked):
per kernel: duration, DRAM bytes read / written (the bench's roofline 'traffic'), DRAM and SM throughput,
tensor-pipe activity, occupancy, registers and the top stall reasons.

  python tools/ncu_summary2.py TAG gpurun_out/round2/full_*.ncu-rep"""
from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys

NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")
KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_hmma_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active": "tma_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__cycles_active.avg": "sm_cycles_active_avg",
    "gpc__cycles_elapsed.max": "cycles_elapsed",
    "smsp__inst_executed.sum": "warp_instructions",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "ns": 1, "us": 1e3, "ms": 1e6, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarize(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?")
    res = {"kernel": name}
    for k, key in KEYS.items():
        if k in d and d[k] not in ("", "n/a"):
            try:
                res[key] = float(d[k].replace(",", "")) * SCALE.get(u.get(k, ""), 1)
            except ValueError:
                pass
    stalls = []
    for k, v in d.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
        if m:
            try:
                stalls.append((float(v), m.group(1)))
            except ValueError:
                pass
    res["top_stalls"] = [f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:5]]
    res["dram_bytes_per_launch"] = res.get("dram_read", 0.0) + res.get("dram_write", 0.0)
    return res


def short(name):
    base = name.split("(")[0].replace("void ", "").strip()
    base = re.sub(r"<.*", "", base)
    return base.split("::")[-1]


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    path = os.path.join("profiles", "ncu_summary.json")
    out = {}
    if os.path.exists(path):  # entries of earlier captures are kept (each names its own tag and capture)
        with open(path) as f:
            out = json.load(f)
        for k, v in out.items():
            if isinstance(v, dict) and "tag" not in v:
                v["tag"] = out.get("tag")
    out.update({"tag": tag, "source": "ncu --set full --clock-control none (one launch per kernel, cold caches)"})
    for rep in reps:
        s = summarize(rep)
        if s:
            s["capture"] = os.path.basename(rep)
            s["tag"] = tag
            out[short(s["kernel"])] = s
            print(short(s["kernel"]), {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()
                                         if k in ("duration_ns", "dram_bytes_per_launch", "dram_pct", "sm_pct",
                                                  "tensor_pct", "issue_pct", "top_stalls")})
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
