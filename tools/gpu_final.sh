#!/bin/bash
# round-end evidence: all GPU tests + smoke, the default bench line (C3 bucketed, sweep), C2, dense C3, C4 and C5
# one-GPU modes, the bench launch list, ncu --set full of the decode and build kernels, compute-sanitizer
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-final}
mkdir -p $OUT
SKIP_NCU=1 SKIP_TESTS=${SKIP_TESTS:-} R2OUT=${R2OUT:-final} bash tools/gpu_full.sh > /dev/null 2>&1
for cfg in C4 C5; do
  timeout 900 python bench.py --config $cfg --steps 200 --warmup 10 --sweep "" --no-cpu-baseline --no-build \
    > $OUT/bench_${cfg}_1.json 2> $OUT/bench_${cfg}_1.err
done
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file $OUT/launches_bench.csv python bench.py --steps 20 --warmup 3 --sweep "" --no-cpu-baseline > /dev/null 2>&1
for k in estimate9 bucket_mark3 select_kernel merge_kernel qencode; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$k python tools/dec_bench.py C3 buckets=1 reps=2 > $OUT/ncu_$k.log 2>&1
done
R2OUT=$(basename $OUT) KS="key_stats_partial r2_partial2 prep_x2 hash_gemm_kernel" bash tools/gpu_ncu_build.sh > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_$tool.log 2>&1
  echo "rc=$?" >> $OUT/sanitize_$tool.log
done
ls -la $OUT
