#!/bin/bash
# round-2 profiling: launch lists (+ optional ncu full captures) of the decode kernels
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-p2}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in ${LSPECS:-"C3:buckets=1" "C3" "C2" "C2:buckets=1"}; do
  tag=${spec//[:=]/_}
  timeout 600 $NCU --metrics $M --clock-control none -c 40 --csv --log-file $OUT/launches_$tag.csv python tools/dec_bench.py ${spec//:/ } reps=2 > /dev/null 2>&1
done
for spec in ${FSPECS:-}; do   # "regex@C3:buckets=1"
  k=${spec%%@*}; w=${spec#*@}; tag=${k}_${w//[:=]/_}
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$tag python tools/dec_bench.py ${w//:/ } reps=2 > $OUT/ncu_$tag.log 2>&1
done
ls -la $OUT
