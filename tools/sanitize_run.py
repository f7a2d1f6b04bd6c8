"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck): every decode kernel generation
(5, 7, 8, 9 and the automatic choice), dense codes and bucketed tables, an emulated 2-shard sequence split
(partial states + merge), at C1-like sizes.  Exits non-zero if an output is non-finite or a status is set.
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2410_16179_b200 as pkg  # noqa: E402
from paper_2410_16179_b200 import binding as B_  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    bad = 0
    for (B, Hq, Hkv, n) in [(1, 4, 1, 2500), (2, 8, 2, 3000)]:
        wl = synth.Workload("san", 990, B=B, Hq=Hq, Hkv=Hkv, n=n, K=10, L=150)
        k, v, q = synth.make_batch(wl)
        W = torch.from_numpy(synth.make_projections(wl.K, wl.L, wl.mips)).to(dev)
        tk, tv, tq = bf(k), bf(v), bf(q)
        for buckets in (False, True):
            mp = pkg.MagicPIG(W, K=wl.K, L=wl.L, buckets=buckets).build(tk)
            ref = None
            for kv in (0, 5, 7, 8, 9):
                B_.set_decode_kernel(kv)
                out = mp.decode(tq, tk, tv)
                torch.cuda.synchronize()
                st = mp.status()
                ok = bool(torch.isfinite(out).all()) and st == 0
                if ref is None:
                    ref = out.clone()
                err = float((out - ref).abs().max())
                print(f"B={B} Hq={Hq} n={n} buckets={buckets} kernel={kv}: finite/status ok={ok} max|diff|={err:.2e}")
                bad += (not ok) or err > 1e-3
            B_.set_decode_kernel(0)
        # emulated 2-shard sequence split: each shard's partial state, then the merge
        n0 = (n // 2 // 1024) * 1024
        parts = []
        mp_full = pkg.MagicPIG(W, K=wl.K, L=wl.L).build(tk)
        for lo, hi in ((0, n0), (n0, n)):
            mps = pkg.MagicPIG(W, K=wl.K, L=wl.L)
            mps._alloc(B, Hkv, hi - lo, dev)
            b = mps.buf
            b.center.copy_(mp_full.buf.center)
            b.r2.copy_(mp_full.buf.r2)
            ks, vs = tk[:, :, lo:hi].contiguous(), tv[:, :, lo:hi].contiguous()
            B_.build_tables(mps.cfg, ks, lo, n, W, b.center, b.r2, b.codes, b.key_norm, mps._ws_build)
            mps.seq_offset, mps.n_global, mps.shape = lo, n, (B, Hkv, hi - lo)
            part = torch.empty((B * Hq, B_.PART), dtype=torch.float32, device=dev)
            mps.decode(tq, ks, vs, partial=part)
            parts.append(part)
        out = torch.empty((B, Hq, 128), dtype=torch.float32, device=dev)
        B_.merge_partials(torch.stack(parts), out)
        full = mp_full.decode(tq, tk, tv)
        torch.cuda.synchronize()
        err = float((out - full).abs().max() / full.abs().max())
        print(f"B={B} Hq={Hq} n={n} 2-shard merge vs unsharded: rel {err:.2e}")
        bad += err > 2e-3
    print("sanitize_run", "FAILED" if bad else "ok")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
