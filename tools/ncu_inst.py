"""Per-source-line executed warp instructions from an ncu report (source page), grouped."""
import csv, io, os, subprocess, sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
hdr = None
cur = None
fname = "?"
inst = defaultdict(float)
text = {}
tot = 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = os.path.basename(row[1])
        continue
    if row[0] == "Line No":
        hdr = row
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    if row[0]:
        cur = (fname, int(row[0]))
        text[cur] = row[1].strip()
        continue
    try:
        v = float(row[ii] or 0)
    except ValueError:
        continue
    inst[cur] += v
    tot += v
print(f"total warp instructions {tot:.0f}  per unit {tot / units:.0f}")
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {v / units:8.0f} {k[0]}:{k[1]:<5d} {text.get(k, '')[:80]}")
