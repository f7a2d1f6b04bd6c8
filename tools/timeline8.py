"""Per-CTA timeline of the tcgen05 estimator (decode kernel 8): python tools/timeline8.py C3 [buckets=1]"""
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

PH = ["start", "prefix", "prod_t0", "prod_last", "mma_t0", "cmp_l0", "cmp_end", "end"]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    wl = synth.CONFIGS[name]
    buckets = 0
    for a_ in sys.argv[2:]:
        k_, v_ = a_.split("=")
        if k_ == "buckets":
            buckets = int(v_)
        else:
            wl = dataclasses.replace(wl, **{k_: int(v_)})
    B_.set_decode_kernel(8)
    dev = torch.device("cuda:0")
    k, v, q = synth.make_batch(wl, threads=8)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    tk, tv, tq = bf(k), bf(v), bf(q)
    tW = torch.from_numpy(W).to(dev)
    reps = []
    for r in range(3):
        kr = tk if r == 0 else tk.clone()
        vr = tv if r == 0 else tv.clone()
        reps.append((pkg.MagicPIG(tW, K=wl.K, L=wl.L, buckets=bool(buckets)).build(kr), kr, vr))
    mp = reps[0][0]
    ws = mp.decode_workspace(wl.B, wl.Hq, wl.Hkv, wl.n, dev)
    out = torch.empty((wl.B, wl.Hq, 128), dtype=torch.float32, device=dev)
    tl = torch.zeros((148 * 8 * 16 * 2,), dtype=torch.int64, device=dev)
    for it in range(7):
        m_, k_, v_ = reps[it % 3]
        rows = B_.debug_decode_timeline(mp.cfg, tq, m_.buf.tables if buckets else m_.buf.codes, m_.buf.center,
                                        m_.buf.key_norm, k_, v_, tW, out, tl, ws, buckets=bool(buckets))
        torch.cuda.synchronize()
    t = tl[:rows * 16].view(rows, 16).cpu().numpy()
    t0 = t[:, 0][t[:, 0] > 0].min()
    print(f"{name} buckets={buckets}: CTAs {rows}")
    for i, nm in enumerate(PH):
        col = t[:, i]
        m = col > 0
        if m.sum() == 0:
            continue
        x = (col[m] - t0) / 1e3
        print(f"  {nm:9s} n={m.sum():4d}  min {x.min():7.2f}  med {np.median(x):7.2f}  max {x.max():7.2f} us")
    print("  tiles per CTA: mean %.1f max %d" % (t[:, 8].mean(), t[:, 8].max()))
    for i, nm in zip(range(9, 16), ["wait_full", "wait_logits", "wait_hashed", "wait_pv", "ph0_issueK+waits",
                                    "ph_a_transform", "ph_bc_pv+soft"]):
        print(f"  {nm:12s} med {np.median(t[:, i]) / 1e3:7.2f} us  max {t[:, i].max() / 1e3:7.2f} us (compute warp 0)")


if __name__ == "__main__":
    main()
