#!/bin/bash
# A/B of two library builds (MAGICPIG_LIB) and dbg variants in ONE call, interleaved, C3 + C2
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-libab}
mkdir -p $OUT
for rep in 1 2; do
  for v in base cur5 cur295; do
    case $v in
      base) L=$PWD/ablib/libmagicpig_base.so; K=5;;
      cur5) L=""; K=5;;
      cur295) L=""; K=295;;
    esac
    echo "== $v rep $rep" >> $OUT/dec.log
    MAGICPIG_LIB=$L timeout 200 python tools/dec_bench.py C3 reps=2 kernel=$K >> $OUT/dec.log 2>&1
    MAGICPIG_LIB=$L timeout 100 python tools/dec_bench.py C2 kernel=$K >> $OUT/dec.log 2>&1
  done
done
