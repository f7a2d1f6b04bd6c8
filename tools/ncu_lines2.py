"""Per CUDA source line: warp-stall samples, instructions executed and top stall reasons
(from ncu --page source --csv --print-source cuda,sass line-aggregate rows).

  python tools/ncu_lines2.py report.ncu-rep [kernel_regex] [top]
"""
from __future__ import annotations

import csv
import io
import os
import subprocess
import sys

NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "."
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    rows, hdr, fname = [], None, "?"
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = os.path.basename(row[1])
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0] or len(row) < len(hdr):
            continue
        d = dict(zip(hdr, row))
        try:
            s, ins = float(row[4] or 0), float(row[7] or 0)
        except ValueError:
            continue
        st = sorted(((h[6:], float(row[i] or 0)) for i, h in enumerate(hdr[:len(row)])
                     if h.startswith("stall_") and "Not Issued" not in h and (row[i] or "0") not in ("0", "-")),
                    key=lambda kv: -kv[1])[:3]
        rows.append((s, ins, fname, row[0], row[1].strip(), st))
    ts = sum(r[0] for r in rows) or 1
    ti = sum(r[1] for r in rows) or 1
    print(f"total samples {ts:.0f}, instructions {ti:.3e}")
    for s, ins, f, ln, txt, st in sorted(rows, key=lambda r: -r[0])[:top]:
        rt = ", ".join(f"{k}={v:.0f}" for k, v in st)
        print(f"{100 * s / ts:5.1f}% smp {100 * ins / ti:5.1f}% ins {f}:{ln:<5s} {txt[:60]:60s} [{rt}]")


if __name__ == "__main__":
    main()
