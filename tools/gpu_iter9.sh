#!/bin/bash
# one iteration on kernel 9: bench stage timings (C3 buckets), the k9 parity subset, optional ncu capture
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-it9}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py --kernel 9 --steps 300 --sweep "" --no-cpu-baseline --no-build --e2e-steps 50 ${BARGS:-} > $OUT/bench_k9.json 2> $OUT/bench_k9.err
python -c "
import json; d=json.load(open('$OUT/bench_k9.json'))
print('STEP', round(d['ms_per_step']*1e3,2), {k: round(v['us'],2) for k, v in d['kernels'].items()}, round(d['roofline']['frac'],3))"
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_append.py -k "k9 or 9" -x -q > $OUT/pytest_k9.log 2>&1; echo "rc=$?" >> $OUT/pytest_k9.log
  tail -n 3 $OUT/pytest_k9.log
fi
if [ -n "$NCUK" ]; then
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$NCUK -s 3 -c 1 -o $OUT/full_$NCUK python tools/dec_bench.py C3 buckets=1 kernel=9 reps=2 > $OUT/ncu.log 2>&1
fi
