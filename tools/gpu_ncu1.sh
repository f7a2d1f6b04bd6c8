#!/bin/bash
# one ncu --set full capture per "kernel_regex@spec" in FSPECS (dec_bench workload)
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-n1}
mkdir -p $OUT
for spec in ${FSPECS}; do
  k=${spec%%@*}; w=${spec#*@}; tag=${k}_${w//[:=]/_}
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$tag python tools/dec_bench.py ${w//:/ } reps=2 > $OUT/ncu_$tag.log 2>&1
done
ls $OUT
