#!/bin/bash
# graph-timed stage combinations for library variants: VARIANTS="base bm1"
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-stages}
mkdir -p $OUT
for v in ${VARIANTS:-base}; do
  L=""; [ "$v" != "base" ] && L=$PWD/ablib/$v/libmagicpig.so
  echo -n "$v " >> $OUT/st.txt
  MAGICPIG_LIB=$L timeout 600 python tools/stage_times.py ${SARGS:-C3} >> $OUT/st.txt 2>> $OUT/err.txt
done
cat $OUT/st.txt
