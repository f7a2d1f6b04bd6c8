#!/bin/bash
# kernel-9 A/B: C3 estimator timings kernel 7 vs 9, then the k9 parity subset
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-k9}
mkdir -p $OUT
for kv in 7 9; do
  for spec in ${SPECS:-"C3 buckets=1" "C3" "C2 buckets=1"}; do
    timeout 300 python tools/dec_bench.py $spec kernel=$kv reps=2 >> $OUT/ab.jsonl 2>> $OUT/ab.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_append.py -k "k9 or 9" -x -q > $OUT/pytest_k9.log 2>&1; echo "rc=$?" >> $OUT/pytest_k9.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "9" > $OUT/pytest_full9.log 2>&1; echo "rc=$?" >> $OUT/pytest_full9.log
ls -la $OUT
