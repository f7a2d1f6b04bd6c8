"""Graph-timed decode stages at a bench config (kernel 9 unless kernel=N): which part of the step is on
the critical path when the kernels are chained with PDL.
  python tools/stage_times.py [C3] [kernel=9] [path=buckets]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2410_16179_b200 import binding as B_  # noqa: E402

args = dict(a.split("=") for a in sys.argv[2:])
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B_.set_decode_kernel(int(args.get("kernel", 9)))
path = args.get("path", "buckets")
dev = torch.device("cuda:0")
wl = synth.CONFIGS[name]
rw = bench.rank_work(wl, bench.MODES[name], 0, 1)
k, v, q = bench.make_rank_inputs(rw, os.cpu_count() or 1)
tW = torch.from_numpy(synth.make_projections(wl.K, wl.L, wl.mips)).to(dev)
R = 2
reps = bench.Replicas(rw, path, dev, R, tW, k, v, q)
cfg, ws = reps.cfg, reps.ws
n = rw.n
out = torch.empty((rw.B, rw.Hq, 128), dtype=torch.float32, device=dev)


def stage(bits, enc=False):
    def fn(r):
        if enc:
            B_.encode_queries(cfg, reps.qs[r], tW, ws)
        B_.debug_decode_stage(cfg, bits, reps.qs[r], reps.codes(r), reps.tables(r), reps.mps[r].buf.center,
                              reps.mps[r].buf.key_norm, reps.ks[r], reps.vs[r], ws, out=out)
    return fn


def enc(r):
    B_.encode_queries(cfg, reps.qs[r], tW, ws)


res = {"encode": bench._graph_time(enc, R, 64)}
for nm, bits, e in (("query", 1, False), ("select", 2, False), ("estimate", 4, False), ("query+select", 3, False),
                    ("select+estimate", 6, False), ("decode", 7, False), ("step", 7, True),
                    ("encode+query", 1, True)):
    res[nm] = bench._graph_time(stage(bits, e), R, 64)
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
