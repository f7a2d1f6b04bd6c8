#!/bin/bash
# ncu --set full of the bucketed Query kernel (bucket_mark3) at C3 on the current build
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-bm3}
mkdir -p $OUT
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:bucket_mark3 -s 3 -c 1 \
  -o $OUT/full_bucket_mark3 python tools/dec_bench.py C3 buckets=1 reps=2 > $OUT/ncu_bucket_mark3.log 2>&1
echo "rc=$?" >> $OUT/ncu_bucket_mark3.log
ls -la $OUT
