"""Per-CTA phase timeline of one decode step (debug ABI), C2 by default.
Prints, per phase, the distribution over CTAs of (stamp - kernel's first start)."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2410_16179_b200 as pkg  # noqa: E402
from paper_2410_16179_b200 import binding as B_  # noqa: E402

PH = ["start", "gdc_wait", "qmasks", "scan", "cl_comb", "compact", "gather", "cta_part", "cl_merge", "umerge0",
      "end"]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    wl = synth.CONFIGS[name]
    dev = torch.device("cuda:0")
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    tk, tv, tq = bf(k), bf(v), bf(q)
    tW = torch.from_numpy(W).to(dev)
    mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L).build(tk)
    ws = mp.decode_workspace(wl.B, wl.Hq, wl.Hkv, wl.n, dev)
    out = torch.empty((wl.B, wl.Hq, 128), dtype=torch.float32, device=dev)
    tl = torch.zeros((100000 * 16,), dtype=torch.int64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    res = []
    for it in range(6):
        flush.zero_()
        grid = B_.debug_decode_timeline(mp.cfg, tq, mp.buf.codes, mp.buf.center, mp.buf.key_norm, tk, tv, tW, out,
                                        tl, ws)
        torch.cuda.synchronize()
        t = tl[:grid * 32].view(grid, 32).cpu().numpy().astype(np.int64)
        res.append(t)
    t = res[-1]
    t0 = t[:, 0][t[:, 0] > 0].min()
    print(f"{name}: {t.shape[0]} CTAs")
    for p, nm in enumerate(PH):
        col = t[:, p]
        col = col[col > 0] - t0
        if len(col) == 0:
            continue
        print(f"{p:2d} {nm:9s} n={len(col):5d}  min={col.min()/1e3:7.2f}  med={np.median(col)/1e3:7.2f}  "
              f"p90={np.percentile(col, 90)/1e3:7.2f}  max={col.max()/1e3:7.2f} us")
    print("gather sub-phases (cycles, median / max over CTAs): ")
    for p, nm in zip(range(11, 15), ["rows_wait", "x+mma", "z+max", "accum"]):
        col = t[:, p]
        print(f"   {nm:10s} med={np.median(col):8.0f} max={col.max():8.0f}")
    m = t[:, 17] > 0
    if m.any():
        print("unit merge (cycles since start, median / max over merging CTAs):")
        for p, nm in zip(range(17, 20), ["ms_staged", "M_S", "done"]):
            print(f"   {nm:10s} med={np.median(t[m, p]):8.0f} max={t[m, p].max():8.0f}")
    # per-phase durations (median over CTAs)
    print("phase durations (median over CTAs, us):")
    for p in range(1, 9):
        m = (t[:, p] > 0) & (t[:, p - 1] > 0)
        if m.any():
            print(f"   {PH[p-1]:>9s} -> {PH[p]:9s}: {np.median(t[m, p] - t[m, p-1])/1e3:7.2f}  max {np.max(t[m, p] - t[m, p-1])/1e3:7.2f}")


if __name__ == "__main__":
    main()
