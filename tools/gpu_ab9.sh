#!/bin/bash
# interleaved A/B of library builds on the kernel-9 bench stage timings: VARIANTS="base pf1 slut0"
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-ab9}
mkdir -p $OUT
for rep in 1 2; do
  for v in ${VARIANTS:-base}; do
    L=""; [ "$v" != "base" ] && L=$PWD/ablib/$v/libmagicpig.so
    MAGICPIG_LIB=$L timeout 600 python bench.py --kernel ${KV:-9} --steps 300 --sweep "${SWEEP:-}" --no-cpu-baseline --no-build --e2e-steps 20 ${BARGS:-} > $OUT/b.json 2>> $OUT/err.txt
    python -c "
import json; d=json.load(open('$OUT/b.json'))
print('$v', 'rep$rep', 'step', round(d['ms_per_step']*1e3,2), {k: round(v['us'],2) for k, v in d['kernels'].items()}, [(s['n'], s['B'], round(s['step_us'], 1), {k: round(v['us'], 1) for k, v in s['kernels'].items()}) for s in (d.get('context_sweep') or [])])" >> $OUT/ab.txt
  done
done
cat $OUT/ab.txt
