"""Build one index (default C2) -- for profiling the build kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2410_16179_b200 as pkg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
wl = synth.CONFIGS[name]
k, v, q = synth.make_batch(wl)
W = synth.make_projections(wl.K, wl.L, wl.mips)
tk = torch.from_numpy(k.view(np.int16)).view(torch.bfloat16).cuda()
mp = pkg.MagicPIG(torch.from_numpy(W).cuda(), K=wl.K, L=wl.L)
for _ in range(3):
    mp.build(tk)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
mp.build(tk)
e.record()
torch.cuda.synchronize()
flops = 2.0 * wl.B * wl.Hkv * wl.n * (128 + wl.mips) * wl.K * wl.L
print(f"{name}: build {s.elapsed_time(e)*1e3:.1f} us, hash flops {flops/1e9:.1f} GFLOP, status {mp.status('build')}")
