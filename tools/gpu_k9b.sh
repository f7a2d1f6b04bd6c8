#!/bin/bash
# kernel 9 stage timings through the bench + ncu full capture of estimate9 at C3 buckets
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-k9b}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
for kv in ${KVS:-9 7}; do
  timeout 600 python bench.py --kernel $kv --steps 300 --sweep "" --no-cpu-baseline --no-build --e2e-steps 50 > $OUT/bench_k$kv.json 2> $OUT/bench_k$kv.err
done
for spec in ${FSPECS:-"estimate9_kernel@C3:buckets=1:kernel=9"}; do
  k=${spec%%@*}; w=${spec#*@}; tag=${k}_${w//[:=]/_}
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$tag python tools/dec_bench.py ${w//:/ } reps=2 > $OUT/ncu_$tag.log 2>&1
done
ls -la $OUT
