#!/bin/bash
# Round-2 evidence run: GPU tests, the default bench line (C3, bucketed) with its sweep, the ncu launch list of
# the bench command, ncu --set full captures of the dominant kernels, compute-sanitizer on small decodes.
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-round2}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err
  timeout 900 python bench.py --path dense --sweep "" --no-cpu-baseline --no-build > $OUT/bench_dense.json 2> $OUT/bench_dense.err
  timeout 900 python bench.py --config C2 --sweep "" --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
fi
if [ -z "$SKIP_NCU" ]; then
  timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 20 --warmup 3 --sweep "" --no-cpu-baseline > /dev/null 2>&1
  for spec in ${FSPECS:-"estimate_kernel@C3:buckets=1" "bucket_mark@C3:buckets=1" "select_kernel@C3:buckets=1" "scan6@C3" "merge_kernel@C3:buckets=1" "qencode@C3:buckets=1" "decode5@C2"}; do
    k=${spec%%@*}; w=${spec#*@}; tag=${k}_${w//[:=]/_}
    timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$tag python tools/dec_bench.py ${w//:/ } reps=2 > $OUT/ncu_$tag.log 2>&1
  done
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:hash_gemm -c 1 -o $OUT/full_hash_gemm_C3 python -c "
import numpy as np, torch, synth, paper_2410_16179_b200 as pkg
wl = synth.CONFIGS['C3']; dev = torch.device('cuda:0')
k, v, q = synth.make_batch(wl, threads=8)
tk = torch.from_numpy(k.view(np.int16)).view(torch.bfloat16).to(dev)
W = torch.from_numpy(synth.make_projections(wl.K, wl.L, wl.mips)).to(dev)
pkg.MagicPIG(W, K=wl.K, L=wl.L).build(tk); torch.cuda.synchronize()" > $OUT/ncu_hash_gemm.log 2>&1
fi
if [ -z "$SKIP_SAN" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_$tool.log 2>&1
    echo "rc=$?" >> $OUT/sanitize_$tool.log
  done
fi
ls -la $OUT
