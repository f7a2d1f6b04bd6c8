#!/bin/bash
# round-2 GPU iteration script: parity (v6 path + buckets) + decode micro-bench
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-r2}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_buckets.py -m gpu -x -q -k "${PYTEST_K:-not k5}" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
for spec in ${SPECS:-"C2" "C2:buckets=1" "C3" "C3:buckets=1"}; do
  timeout 300 python tools/dec_bench.py ${spec//:/ } >> $OUT/dec.jsonl 2>> $OUT/dec.err
done
tail -3 $OUT/pytest.log; cat $OUT/dec.jsonl
