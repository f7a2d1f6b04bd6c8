#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-v5}
mkdir -p $OUT
timeout 120 python tools/dec_bench.py C2 > $OUT/dec.log 2>&1
echo "dec exit $?" >> $OUT/dec.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 120 > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 120 python tools/timeline.py C2 > $OUT/timeline_c2.log 2>&1
timeout 120 python tools/timeline.py C2 kernel=25 > $OUT/timeline_c2_nopf.log 2>&1
timeout 300 python tools/timeline.py C3 > $OUT/timeline_c3.log 2>&1
timeout 300 python tools/dec_bench.py C2 n=131072 >> $OUT/dec.log 2>&1
timeout 600 python tools/dec_bench.py C3 reps=2 >> $OUT/dec.log 2>&1
