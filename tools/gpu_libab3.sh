#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-libab}
mkdir -p $OUT
for v in base e960 d8a9 cur base e960; do
  case $v in
    cur) L="";;
    *) L=$PWD/ablib/libmagicpig_$v.so;;
  esac
  echo "== $v" >> $OUT/dec.log
  MAGICPIG_LIB=$L timeout 200 python tools/dec_bench.py C3 reps=2 >> $OUT/dec.log 2>&1
done
