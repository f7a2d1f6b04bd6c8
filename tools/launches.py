"""Summarise ncu launch-list CSVs: per kernel name, mean duration (us) and DRAM MB per launch.

  python tools/launches.py gpurun_out/p2/launches_*.csv
"""
import csv
import sys
from collections import defaultdict

for fn in sys.argv[1:]:
    rows = list(csv.reader(open(fn)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = defaultdict(list)
    ids = sorted(data)
    for (i, k) in ids[len(ids) // 2:]:  # second half: warm
        agg[k.split("(")[0][:60]].append(data[(i, k)])
    print(fn)
    for k, ms in agg.items():
        t = sum(m.get("gpu__time_duration.sum", 0) for m in ms) / len(ms) / 1e3
        rd = sum(m.get("dram__bytes_read.sum", 0) for m in ms) / len(ms) / 1e6
        wr = sum(m.get("dram__bytes_write.sum", 0) for m in ms) / len(ms) / 1e6
        print(f"  {k:60s} n={len(ms):3d} {t:9.2f} us  read {rd:8.2f} MB  write {wr:6.2f} MB  {(rd + wr) / max(t, 1e-9):6.2f} TB/s")
