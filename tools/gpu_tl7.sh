#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-tl7}
mkdir -p $OUT
for spec in ${SPECS:-"C2" "C2:buckets=1" "C3:buckets=1"}; do
  timeout 300 python tools/timeline7.py ${spec//:/ } >> $OUT/tl.txt 2>&1
done
cat $OUT/tl.txt
