#!/bin/bash
# new tests (full-size units, append loop, adversarial fix-up), multi-rank bench modes on one GPU (gloo), harness
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-r2e}
mkdir -p $OUT
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_append.py tests/test_gpu_parity.py -m gpu -q -x \
  -k "${PYTEST_K:-fullsize or append or sharding or all_units or cancellation}" > $OUT/pytest_new.log 2>&1
echo "rc=$?" >> $OUT/pytest_new.log
for cfg in C4 C5; do
  MAGICPIG_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config $cfg --steps 50 --warmup 5 --sweep "" \
    --no-cpu-baseline --no-build > $OUT/bench_${cfg}_2rank.json 2> $OUT/bench_${cfg}_2rank.err
  timeout 900 python bench.py --config $cfg --steps 200 --warmup 10 --sweep "" --no-cpu-baseline --no-build \
    > $OUT/bench_${cfg}_1.json 2> $OUT/bench_${cfg}_1.err
done
timeout 1200 python tools/estimator_quality.py --n 16384 --units 2 --out $OUT/estimator_quality.json > $OUT/eq.log 2>&1
tail -3 $OUT/pytest_new.log; tail -2 $OUT/*.err | head -30; cut -c1-300 $OUT/bench_*.json; tail -30 $OUT/eq.log
