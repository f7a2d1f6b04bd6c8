#!/bin/bash
# A/B of library builds (MAGICPIG_LIB) in ONE call, interleaved: VARIANTS="base nw10"
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-libab7}
mkdir -p $OUT
for rep in 1 2; do
  for v in ${VARIANTS:-base}; do
    L=""; [ "$v" != "base" ] && L=$PWD/ablib/$v/libmagicpig.so
    for spec in ${SPECS:-"C3:buckets=1" "C2"}; do
      echo -n "$v rep$rep $spec " >> $OUT/ab.txt
      MAGICPIG_LIB=$L timeout 300 python tools/dec_bench.py ${spec//:/ } 2>>$OUT/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kernel %.2f step %.2f' % (d['kernel_us'], d['step_us']))" >> $OUT/ab.txt
    done
  done
done
cat $OUT/ab.txt
