#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-libab}
mkdir -p $OUT
for v in keep new keep new; do
  case $v in
    new) L="";;
    *) L=$PWD/ablib/libmagicpig_$v.so;;
  esac
  echo "== $v" >> $OUT/dec.log
  MAGICPIG_LIB=$L timeout 200 python tools/dec_bench.py C3 reps=2 >> $OUT/dec.log 2>&1
  MAGICPIG_LIB=$L timeout 100 python tools/dec_bench.py C2 >> $OUT/dec.log 2>&1
  MAGICPIG_LIB=$L timeout 100 python tools/dec_bench.py C2 n=131072 reps=2 >> $OUT/dec.log 2>&1
done
timeout 400 python -m pytest tests/test_gpu_buckets.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 200 > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
