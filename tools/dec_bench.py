"""Decode kernel micro-benchmark: kernel-only and encode+decode step times,
algorithmic bytes and roofline fraction, for a config (optionally with n / B
overridden).  For iteration; bench.py is the contract.

  python tools/dec_bench.py C2 [n=65536] [B=8] [reps=4]
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2410_16179_b200 as pkg  # noqa: E402
from paper_2410_16179_b200 import binding as B_  # noqa: E402


def run(name, R=4, G_STEPS=64, buckets=0, **over):
    wl = dataclasses.replace(synth.CONFIGS[name], **over)
    dev = torch.device("cuda:0")
    k, v, q = synth.make_batch(wl)
    W = synth.make_projections(wl.K, wl.L, wl.mips)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    tk, tv, tq, tW = bf(k), bf(v), bf(q), torch.from_numpy(W).to(dev)
    del k, v
    mps, ks, vs = [], [], []
    for r in range(R):
        kr = tk if r == 0 else tk.clone()
        vr = tv if r == 0 else tv.clone()
        mp = pkg.MagicPIG(tW, K=wl.K, L=wl.L, mips=wl.mips, buckets=bool(buckets)).build(kr)
        mp.release_build_workspace()
        mps.append(mp), ks.append(kr), vs.append(vr)
    cfg = mps[0].cfg
    n, Bn, Hq, Hkv = wl.n, wl.B, wl.Hq, wl.Hkv
    ws = B_.new_workspace(B_.decode_workspace_bytes(cfg, Bn, Hq, Hkv, n), dev)
    out = torch.empty((Bn, Hq, 128), dtype=torch.float32, device=dev)
    nw = (n + 31) // 32
    smask = torch.zeros((Bn, Hq, nw), dtype=torch.int32, device=dev)
    scount = torch.zeros((Bn, Hq), dtype=torch.int32, device=dev)
    mps[0]._ws_dec = ws
    mps[0].decode(tq, ks[0], vs[0], out=out, s_count=scount, s_mask=smask)
    torch.cuda.synchronize()
    sm = smask.cpu().numpy().view(np.uint32).reshape(Bn, Hkv, wl.G, nw)
    union = np.bitwise_or.reduce(sm, axis=2)
    n_union = int(np.unpackbits(union.view(np.uint8)).sum())
    nT = min(n, wl.sink + wl.local)
    KL = wl.K * wl.L
    alg = Bn * Hkv * (n - nT) * KL / 8 + (n_union + Bn * Hkv * nT) * 512 + n_union * 4 + Bn * Hq * (256 + KL / 8) \
        + Bn * Hkv * 512

    def kern(r):
        if buckets:
            B_.decode_buckets_encoded(cfg, tq, mps[r].buf.tables, mps[r].buf.center, mps[r].buf.key_norm, ks[r], vs[r],
                                      0, n, ws, out=out)
        else:
            B_.decode_encoded(cfg, tq, mps[r].buf.codes, mps[r].buf.center, mps[r].buf.key_norm, ks[r], vs[r], 0, n,
                              ws, out=out)

    def step(r):
        B_.encode_queries(cfg, tq, tW, ws)
        kern(r)

    res = {}
    for nm, fn in (("kernel", kern), ("step", step)):
        for r in range(R):
            fn(r)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(G_STEPS):
                fn(i % R)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / G_STEPS)
        res[nm + "_us"] = float(np.median(ts))
    if buckets:  # codes term -> the ids of the query's buckets + offsets + S bitmaps (write + read)
        qc = torch.zeros((Bn, Hq, wl.L), dtype=torch.int16, device=dev)
        B_.query_codes(cfg, tq, tW, qc, ws)
        qc = qc.cpu().numpy().view(np.uint16).astype(np.int64)
        nb = 1 << wl.K
        per = B_.bucket_tables_words(cfg, 1, 1, n)  # words per unit (16-bit ids when n <= 65536)
        tabs = mps[0].buf.tables.cpu().numpy()
        ids_read = 0
        for b in range(Bn):
            for hq in range(Hq):
                u = b * Hkv + hq // wl.G
                offs = tabs[u * per:u * per + wl.L * (nb + 1)].reshape(wl.L, nb + 1)
                c = qc[b, hq]
                ids_read += int((offs[np.arange(wl.L), c + 1] - offs[np.arange(wl.L), c]).sum())
        alg = alg - Bn * Hkv * (n - nT) * KL / 8 + ids_read * (2 if n <= 65536 else 4) + Bn * Hq * wl.L * 8 + 2 * Bn * Hq * ((n + 31) // 32) * 4
        res["ids_read"] = ids_read
    res.update(config=name, n=n, B=Bn, K=wl.K, L=wl.L, alg_MB=alg / 1e6, buckets=buckets,
               sampled=float(scount.float().mean()) / max(n - nT, 1), union=n_union,
               GBs=alg / res["kernel_us"] / 1e3, frac=alg / res["kernel_us"] / 1e3 / 6545.0,
               status=B_.workspace_status(ws))
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    kw = {}
    R = 4
    for a in sys.argv[2:]:
        key, val = a.split("=")
        if key == "reps":
            R = int(val)
        elif key == "buckets":
            kw["buckets"] = int(val)
        elif key == "kernel":
            B_.set_decode_kernel(int(val))
        else:
            kw[key] = int(val)
    run(name, R=R, **kw)
