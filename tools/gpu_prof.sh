#!/bin/bash
# decode micro-bench sweep + ncu source-level capture of the decode kernel
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
timeout 300 python tools/dec_bench.py C2 > $OUT/dec_c2.log 2>&1
for nn in 4096 8192 32768 65536 131072; do timeout 200 python tools/dec_bench.py C2 n=$nn >> $OUT/dec_ctx.log 2>&1; done
timeout 600 python tools/dec_bench.py C3 reps=2 > $OUT/dec_c3.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"decode_kernel" -s 8 -c 1 \
   -o $OUT/dec_full python tools/dec_bench.py C2 reps=2 > $OUT/ncu_dec.log 2>&1
