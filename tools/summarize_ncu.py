"""Summarise ncu captures into profiles/ (tracked): per-kernel duration, DRAM
bytes, throughput and the top stall reasons.

  python tools/summarize_ncu.py gpurun_out/decode_full.ncu-rep gpurun_out/launches.csv r01
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

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
    "launch__cluster_dim_x": "cluster_x",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
              "ns": 1, "us": 1e3, "ms": 1e6, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1}


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(rep):
    h, units, rows = raw(rep)
    res = defaultdict(list)
    for r in rows:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        rec = {}
        for k, short in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                v *= UNIT_SCALE.get(u.get(k, ""), 1)
                rec[short] = v
        stalls = []
        for k in h:
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(d[k].replace(",", "") or 0), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        rec["top_stalls"] = [s for _, s in sorted(stalls, reverse=True)[:5]]
        res[name].append(rec)
    summary = {}
    for name, recs in res.items():
        agg = {"launches": len(recs)}
        for short in KEYS.values():
            vals = [r[short] for r in recs if short in r]
            if vals:
                agg[short] = sum(vals) / len(vals)
        if "dram_read" in agg:
            agg["dram_bytes_per_launch"] = agg["dram_read"] + agg.get("dram_write", 0.0)
        agg["top_stalls"] = recs[0]["top_stalls"]
        summary[name] = agg
    return summary


def launches(csvfile):
    rows = list(csv.reader(open(csvfile)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    return {k: {"n": len(v), "mean_us": sum(v) / len(v) / 1e3, "share": sum(v) / tot}
            for k, v in sorted(d.items(), key=lambda x: -sum(x[1]))}


def main():
    rep, lcsv, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs("profiles", exist_ok=True)
    s = summarize(rep)
    L = launches(lcsv)
    decode = next((v for k, v in s.items() if "decode5_kernel" in k), None) or \
        next((v for k, v in s.items() if "decode_kernel" in k), None)
    out = {"tag": tag, "kernels": s, "launch_list": L,
           "decode": {"dram_bytes_per_launch": decode.get("dram_bytes_per_launch")} if decode else {}}
    with open("profiles/ncu_summary.json", "w") as f:
        json.dump(out, f, indent=1)
    with open(f"profiles/{tag}_ncu_summary.txt", "w") as f:
        f.write(f"# ncu summary {tag} (from {os.path.basename(rep)}, {os.path.basename(lcsv)})\n\n")
        f.write("## launch list (gpu__time_duration.sum, cold-cache serialised)\n")
        for k, v in L.items():
            f.write(f"{k:40s} n={v['n']:5d} mean={v['mean_us']:9.2f} us share={v['share']*100:5.1f}%\n")
        f.write("\n## --set full per kernel (mean over captured launches)\n")
        for k, v in s.items():
            f.write(f"{k}\n")
            for kk, vv in v.items():
                f.write(f"   {kk}: {vv}\n")
    print(json.dumps(out["decode"]))


if __name__ == "__main__":
    main()
