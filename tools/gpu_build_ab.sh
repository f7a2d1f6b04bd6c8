#!/bin/bash
# A/B of the index-build phase timings (bench 'build' key) over library variants: VARIANTS="base hgu4"
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-bab}
mkdir -p $OUT
for v in ${VARIANTS:-base}; do
  L=""; [ "$v" != "base" ] && L=$PWD/ablib/$v/libmagicpig.so
  MAGICPIG_LIB=$L timeout 600 python bench.py --steps 50 --sweep "" --no-cpu-baseline --e2e-steps 10 > $OUT/b_$v.json 2>> $OUT/err.txt
  python -c "
import json; d=json.load(open('$OUT/b_$v.json'))['build']
print('$v', {k: round(v, 1) for k, v in d.items() if k.endswith('_us') or k in ('hash_tflops', 'tensor_frac')})" >> $OUT/ab.txt
done
cat $OUT/ab.txt
