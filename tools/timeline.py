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
    import dataclasses
    kver = 5
    for a_ in sys.argv[2:]:
        k_, v_ = a_.split('=')
        if k_ == "kernel":
            kver = int(v_)
            continue
        wl = dataclasses.replace(wl, **{k_: int(v_)})
    B_.set_decode_kernel(kver)
    dev = torch.device("cuda:0")
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    tk, tv, tq = bf(k), bf(v), bf(q)
    tW = torch.from_numpy(W).to(dev)
    # warm mode (default): 4 replicas used round-robin, no flush -> the kernel's code is hot in L2 while
    # the data of the measured launch was last touched 3 launches (> L2) ago, as in bench.py.
    # cold mode (flush=1): a 512 MB write before every launch evicts code and data.
    cold = os.environ.get("TL_COLD", "0") == "1"
    R = 1 if cold else 4
    reps = []
    for r in range(R):
        kr = tk if r == 0 else tk.clone()
        vr = tv if r == 0 else tv.clone()
        reps.append((pkg.MagicPIG(tW, K=wl.K, L=wl.L).build(kr), kr, vr))
    mp = reps[0][0]
    ws = mp.decode_workspace(wl.B, wl.Hq, wl.Hkv, wl.n, dev)
    out = torch.empty((wl.B, wl.Hq, 128), dtype=torch.float32, device=dev)
    tl = torch.zeros((200000 * 32,), dtype=torch.int64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    res = []
    for it in range(9 if not cold else 6):
        if cold:
            flush.zero_()
        m_, k_, v_ = reps[it % R]
        grid = B_.debug_decode_timeline(mp.cfg, tq, m_.buf.codes, m_.buf.center, m_.buf.key_norm, k_, v_, tW, out,
                                        tl, ws)
        torch.cuda.synchronize()
        t = tl[:grid * 32].view(grid, 32).cpu().numpy().astype(np.int64)
        res.append(t)
    t = res[-1]
    st = t[:, 0].astype(np.int64)
    st = st - st[st > 0].min()
    print(f"{name}: {t.shape[0]} CTAs; CTA start spread: med {np.median(st)/1e3:.2f} us, max {st.max()/1e3:.2f} us")
    ghz = 1.965
    if kver % 10 == 5:
        names = ["start", "qmasks", "desc0", "batch0", "merge0", "merge1", "gdone", "gdc_wait", "qbw_ld", "sc_bar1",
                 "prod_end"] + [f"scanw{w}" for w in range(8)] + ["m_loaded", "m_comp", "flush0", "atomic"]
        names[10] = "sc_bar2"
        names += ["-"] * 6 + ["b0_rows", "b0_xbar", "b0_z"]
        for p in list(range(1, 23)) + [29, 30, 31]:
            col = t[:, p]
            m = col > 0
            if not m.any():
                continue
            us = (col[m] - 1) / ghz / 1e3 + st[m] / 1e3
            print(f"{p:2d} {names[p]:9s} n={m.sum():5d}  (abs) min={us.min():7.2f}  med={np.median(us):7.2f}  "
                  f"p90={np.percentile(us, 90):7.2f}  max={us.max():7.2f} us")
        print("per-CTA totals (us, median / max):")
        for p, nm in zip(range(23, 29), ["scan: wait codes", "scan: wait desc", "scan: total", "gather: wait desc",
                                          "gather: wait rows", "gather: total"]):
            col = t[:, p].astype(np.float64) / ghz / 1e3
            print(f"   {nm:18s} {np.median(col):8.2f} {col.max():8.2f}")
        return
    for p, nm in enumerate(PH):
        if p == 0:
            continue
        col = t[:, p]
        m = col > 0
        if not m.any():
            continue
        us = (col[m] - 1) / ghz / 1e3 + st[m] / 1e3
        print(f"{p:2d} {nm:9s} n={m.sum():5d}  (abs) min={us.min():7.2f}  med={np.median(us):7.2f}  "
              f"p90={np.percentile(us, 90):7.2f}  max={us.max():7.2f} us")
    print("gather sub-phases (cycles, median / max over CTAs): ")
    for p, nm in zip(range(11, 15), ["rows_wait", "x+mma", "z+max", "accum"]):
        col = t[:, p]
        print(f"   {nm:10s} med={np.median(col):8.0f} max={col.max():8.0f}")
    life = (t[:, 8].astype(np.int64) - 1) / ghz / 1e3
    print(f"CTA lifetime to cl_merge (us): med {np.median(life):.2f}  p90 {np.percentile(life, 90):.2f}  max {life.max():.2f}")
    m = t[:, 17] > 0
    if m.any():
        print("unit merge (cycles since start, median / max over merging CTAs):")
        for p, nm in zip(range(17, 20), ["ms_staged", "M_S", "done"]):
            print(f"   {nm:10s} med={np.median(t[m, p]):8.0f} max={t[m, p].max():8.0f}")
    print("phase durations (median / max over CTAs, us, from SM cycles):")
    for p in range(2, 9):
        m = (t[:, p] > 0) & (t[:, p - 1] > 0)
        if m.any():
            dd = (t[m, p].astype(np.int64) - t[m, p - 1].astype(np.int64)) / ghz / 1e3
            print(f"   {PH[p-1]:>9s} -> {PH[p]:9s}: {np.median(dd):7.2f}  max {dd.max():7.2f}")


if __name__ == "__main__":
    main()
