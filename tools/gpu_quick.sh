#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-q}
mkdir -p $OUT
timeout 120 python tools/dec_bench.py C2 > $OUT/dec.log 2>&1
timeout 300 python tools/dec_bench.py C2 n=131072 >> $OUT/dec.log 2>&1
timeout 600 python tools/dec_bench.py C3 reps=2 >> $OUT/dec.log 2>&1
timeout 120 python tools/timeline.py C2 > $OUT/timeline_c2.log 2>&1
timeout 300 python tools/timeline.py C3 > $OUT/timeline_c3.log 2>&1
