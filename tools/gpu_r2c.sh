#!/bin/bash
# iteration: parity on the default path, decode micro-bench, v7 timelines
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-r2c}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_buckets.py -m gpu -q -x -k "${PYTEST_K:-not k5 and not k6}" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
for spec in ${SPECS:-"C2" "C2:buckets=1" "C3" "C3:buckets=1"}; do
  timeout 300 python tools/dec_bench.py ${spec//:/ } >> $OUT/dec.jsonl 2>> $OUT/dec.err
done
for spec in ${TSPECS:-"C2" "C3:buckets=1"}; do
  timeout 300 python tools/timeline7.py ${spec//:/ } >> $OUT/tl.txt 2>&1
done
tail -3 $OUT/pytest.log; cat $OUT/dec.jsonl; grep -v "slow row" $OUT/tl.txt
