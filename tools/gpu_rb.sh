#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-rb}
mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_buckets.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 200 > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
for bk in 0 1; do
  timeout 120 python tools/dec_bench.py C2 buckets=$bk >> $OUT/dec.log 2>&1
  timeout 120 python tools/dec_bench.py C2 n=131072 reps=2 buckets=$bk >> $OUT/dec.log 2>&1
  timeout 200 python tools/dec_bench.py C3 reps=2 buckets=$bk >> $OUT/dec.log 2>&1
done
timeout 120 python tools/timeline.py C2 > $OUT/timeline_c2.log 2>&1
