#!/bin/bash
# round-2 status run: full GPU test suite + decode micro-bench (v6) at C2/C3, dense and bucketed
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-r2a}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
for spec in ${SPECS:-"C2" "C2:buckets=1" "C3" "C3:buckets=1" "C2:kernel=5" "C3:kernel=5" "C3:buckets=1:kernel=5"}; do
  timeout 300 python tools/dec_bench.py ${spec//:/ } >> $OUT/dec.jsonl 2>> $OUT/dec.err
done
tail -3 $OUT/pytest.log; cat $OUT/dec.jsonl
