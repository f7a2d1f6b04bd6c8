#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-bk}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_buckets.py -m gpu -q -x -p no:cacheprovider --timeout 300 > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
for bk in 1 0; do
  timeout 120 python tools/dec_bench.py C2 buckets=$bk >> $OUT/dec.log 2>&1
  timeout 300 python tools/dec_bench.py C2 n=131072 reps=2 buckets=$bk >> $OUT/dec.log 2>&1
  timeout 600 python tools/dec_bench.py C3 reps=2 buckets=$bk >> $OUT/dec.log 2>&1
done
