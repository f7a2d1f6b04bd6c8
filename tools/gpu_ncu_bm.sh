#!/bin/bash
# ncu --set full of the bucketed Query kernel and the select kernel at C3 (kernel 9 path)
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-bm}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
for k in ${KS:-bucket_mark select_kernel}; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$k python tools/dec_bench.py C3 buckets=1 kernel=9 reps=2 > $OUT/ncu_$k.log 2>&1
done
python - <<'PY' > $OUT/bm_stats.txt 2>&1
# distribution of bucket ids per query head at C3 (how skewed the Query work is)
import numpy as np, torch, synth, paper_2410_16179_b200 as pkg
from paper_2410_16179_b200 import binding as B_
wl = synth.CONFIGS['C3']; dev = torch.device('cuda:0')
k, v, q = synth.make_batch(wl, threads=8)
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
tk, tq = bf(k), bf(q)
W = torch.from_numpy(synth.make_projections(wl.K, wl.L, wl.mips)).to(dev)
mp = pkg.MagicPIG(W, K=wl.K, L=wl.L, mips=wl.mips, buckets=True).build(tk)
ws = B_.new_workspace(B_.decode_workspace_bytes(mp.cfg, wl.B, wl.Hq, wl.Hkv, wl.n), dev)
qc = torch.zeros((wl.B, wl.Hq, wl.L), dtype=torch.int16, device=dev)
B_.query_codes(mp.cfg, tq, W, qc, ws)
qc = qc.cpu().numpy().view(np.uint16).astype(np.int64)
nb = 1 << wl.K; per = wl.L * (nb + 1 + wl.n)
tabs = mp.buf.tables.cpu().numpy()
tot = []
mx = []
for b in range(wl.B):
    for hq in range(wl.Hq):
        u = b * wl.Hkv + hq // wl.G
        offs = tabs[u * per:u * per + wl.L * (nb + 1)].reshape(wl.L, nb + 1)
        c = qc[b, hq]
        sz = offs[np.arange(wl.L), c + 1] - offs[np.arange(wl.L), c]
        tot.append(int(sz.sum())); mx.append(int(sz.max()))
tot = np.array(tot); mx = np.array(mx)
print("ids per head: mean %.0f median %.0f max %d min %d p90 %.0f" % (tot.mean(), np.median(tot), tot.max(), tot.min(), np.percentile(tot, 90)))
print("largest bucket per head: mean %.0f max %d" % (mx.mean(), mx.max()))
print("sorted top 20:", sorted(tot.tolist())[-20:])
PY
cat $OUT/bm_stats.txt
