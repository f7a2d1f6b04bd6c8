#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-v5}
mkdir -p $OUT
timeout 120 python tools/dec_bench.py C2 > $OUT/dec.log 2>&1
timeout 300 python tools/dec_bench.py C2 n=131072 >> $OUT/dec.log 2>&1
timeout 600 python tools/dec_bench.py C3 reps=2 >> $OUT/dec.log 2>&1
timeout 120 python tools/timeline.py C2 > $OUT/timeline_c2.log 2>&1
timeout 300 python tools/timeline.py C3 > $OUT/timeline_c3.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"decode5_kernel" -s 8 -c 1 \
   -o $OUT/dec_c2 python tools/dec_bench.py C2 reps=2 > $OUT/ncu_c2.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"decode5_kernel" -s 4 -c 1 \
   -o $OUT/dec_c3 python tools/dec_bench.py C3 reps=1 > $OUT/ncu_c3.log 2>&1
