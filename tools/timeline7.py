"""Per-warp phase timeline of the v7 estimator (debug ABI): python tools/timeline7.py C2 [buckets=1] [n=...]
Prints, per phase, the distribution over active warps of (stamp - earliest kernel start), in us,
and the slowest warps."""
from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2410_16179_b200 as pkg  # noqa: E402
from paper_2410_16179_b200 import binding as B_  # noqa: E402

PH = ["start", "gdc_wait", "prefix", "plan0", "issue0", "data0", "computed", "flush0", "merge0", "merge1", "end",
      "slabs", "merges"]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    wl = synth.CONFIGS[name]
    buckets = 0
    for a_ in sys.argv[2:]:
        k_, v_ = a_.split("=")
        if k_ == "buckets":
            buckets = int(v_)
        else:
            wl = dataclasses.replace(wl, **{k_: int(v_)})
    dev = torch.device("cuda:0")
    k, v, q = synth.make_batch(wl, threads=8)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    tk, tv, tq = bf(k), bf(v), bf(q)
    tW = torch.from_numpy(W).to(dev)
    R = 3
    reps = []
    for r in range(R):
        kr = tk if r == 0 else tk.clone()
        vr = tv if r == 0 else tv.clone()
        reps.append((pkg.MagicPIG(tW, K=wl.K, L=wl.L, buckets=bool(buckets)).build(kr), kr, vr))
    mp = reps[0][0]
    ws = mp.decode_workspace(wl.B, wl.Hq, wl.Hkv, wl.n, dev)
    out = torch.empty((wl.B, wl.Hq, 128), dtype=torch.float32, device=dev)
    tl = torch.zeros((148 * 8 * 16 * 2,), dtype=torch.int64, device=dev)
    res = []
    for it in range(7):
        m_, k_, v_ = reps[it % R]
        rows = B_.debug_decode_timeline(mp.cfg, tq, m_.buf.tables if buckets else m_.buf.codes, m_.buf.center,
                                        m_.buf.key_norm, k_, v_, tW, out, tl, ws, buckets=bool(buckets))
        torch.cuda.synchronize()
        if it >= 3:
            res.append(tl[:rows * 16].view(rows, 16).cpu().numpy().copy())
    t = res[-1]
    act = t[:, 0] > 0
    t0 = t[act, 0].min()
    print(f"{name} buckets={buckets}: rows {t.shape[0]}, active-stamped {act.sum()}, "
          f"issuing warps {(t[:, 4] > 0).sum()}")
    for i, nm in enumerate(PH[:11]):
        col = t[:, i]
        m = col > 0
        if m.sum() == 0:
            continue
        x = (col[m] - t0) / 1e3
        print(f"  {nm:9s} n={m.sum():5d}  min {x.min():7.2f}  med {np.median(x):7.2f}  max {x.max():7.2f} us")
    print("  slabs per issuing warp: mean %.1f max %d; merges %d" % (t[t[:, 4] > 0, 11].mean(),
                                                                     t[:, 11].max(), t[:, 12].sum()))
    order = np.argsort(-(t[:, 10] - t0) * act)[:5]
    for r in order:
        print("  slow row", r, "cta", r // 8, "warp", r % 8, [(PH[i], round((t[r, i] - t0) / 1e3, 2)) for i in range(11)
                                                             if t[r, i] > 0], "slabs", t[r, 11], "merges", t[r, 12])


if __name__ == "__main__":
    main()
