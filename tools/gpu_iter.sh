#!/bin/bash
# quick iteration: gpu parity tests + decode micro-bench + timelines
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-iter}
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python tools/dec_bench.py C2 > $OUT/dec.log 2>&1
timeout 300 python tools/dec_bench.py C2 n=131072 >> $OUT/dec.log 2>&1
timeout 600 python tools/dec_bench.py C3 reps=2 >> $OUT/dec.log 2>&1
timeout 300 python tools/timeline.py C2 > $OUT/timeline_c2.log 2>&1
timeout 300 python tools/timeline.py C3 > $OUT/timeline_c3.log 2>&1
