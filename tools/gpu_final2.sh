#!/bin/bash
# round-end evidence on the final build: GPU tests + smoke, bench default (C3 bucketed + sweep), C2, C4, C5,
# the bench launch list and ncu --set full of the estimator, the Query kernel and the hash GEMM
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-final2}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --config C2 --sweep "" --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for cfg in C4 C5; do
  timeout 900 python bench.py --config $cfg --steps 200 --warmup 10 --sweep "" --no-cpu-baseline --no-build \
    > $OUT/bench_${cfg}_1.json 2> $OUT/bench_${cfg}_1.err
done
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file $OUT/launches_bench.csv python bench.py --steps 20 --warmup 3 --sweep "" --no-cpu-baseline > /dev/null 2>&1
for k in estimate9 bucket_mark3 merge_kernel; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$k python tools/dec_bench.py C3 buckets=1 reps=2 > $OUT/ncu_$k.log 2>&1
done
R2OUT=$(basename $OUT) KS="hash_gemm_kernel" bash tools/gpu_ncu_build.sh > /dev/null 2>&1
ls -la $OUT
