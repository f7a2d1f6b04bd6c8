"""Aggregate ncu warp-stall samples per CUDA source line (from --page source
--print-source cuda,sass) and print the hottest lines with their top stall reasons.

  python tools/ncu_lines.py report.ncu-rep [kernel_regex] [top]
"""
from __future__ import annotations

import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "decode_kernel"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    per_line = defaultdict(float)
    reasons = defaultdict(lambda: defaultdict(float))
    text = {}
    fname = "?"
    hdr = None
    cur = None
    total = 0.0
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = os.path.basename(row[1])
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < len(hdr):
            continue
        if row[0]:
            cur = (fname, int(row[0]))
            text[cur] = row[1].strip()
            continue
        try:
            s = float(row[4] or 0)
        except ValueError:
            continue
        total += s
        per_line[cur] += s
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and i < len(row):
                try:
                    reasons[cur][h[6:]] += float(row[i] or 0)
                except ValueError:
                    pass
    print(f"total samples {total:.0f}")
    for key, s in sorted(per_line.items(), key=lambda kv: -kv[1])[:top]:
        rs = sorted(reasons[key].items(), key=lambda kv: -kv[1])[:3]
        rtxt = ", ".join(f"{k}={v:.0f}" for k, v in rs if v > 0)
        print(f"{100 * s / max(total, 1):5.1f}% {key[0]}:{key[1]:<5d} {text.get(key, '')[:70]:70s} [{rtxt}]")


if __name__ == "__main__":
    main()
