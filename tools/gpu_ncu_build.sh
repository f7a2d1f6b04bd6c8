#!/bin/bash
# ncu --set full of the build kernels at C3 (one launch each)
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-nb}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
cat > tools/_build_c3.py <<'PY'
import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, paper_2410_16179_b200 as pkg
wl = synth.CONFIGS['C3']; dev = torch.device('cuda:0')
k, v, q = synth.make_batch(wl, threads=8)
tk = torch.from_numpy(k.view(np.int16)).view(torch.bfloat16).to(dev)
W = torch.from_numpy(synth.make_projections(wl.K, wl.L, wl.mips)).to(dev)
pkg.MagicPIG(W, K=wl.K, L=wl.L).build(tk); torch.cuda.synchronize()
PY
for k in ${KS:-key_stats_partial r2_partial prep_x hash_gemm_kernel}; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -c 1 -o $OUT/full_$k python tools/_build_c3.py > $OUT/ncu_$k.log 2>&1
done
ls -la $OUT
