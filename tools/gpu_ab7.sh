#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-ab7}
mkdir -p $OUT
for spec in ${SPECS:-"C3:buckets=1:kernel=7" "C3:buckets=1:kernel=17" "C2:buckets=1:kernel=7" "C2:buckets=1:kernel=17"}; do
  timeout 300 python tools/dec_bench.py ${spec//:/ } >> $OUT/dec.jsonl 2>> $OUT/dec.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in ${LSPECS:-"C3:buckets=1:kernel=7" "C3:buckets=1:kernel=17"}; do
  tag=${spec//[:=]/_}
  timeout 600 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -c 40 --csv --log-file $OUT/launches_$tag.csv python tools/dec_bench.py ${spec//:/ } reps=2 > /dev/null 2>&1
  python tools/launches.py $OUT/launches_$tag.csv >> $OUT/launches.txt
done
cat $OUT/dec.jsonl | cut -c1-200; cat $OUT/launches.txt
