#!/bin/bash
# full evidence run: all GPU tests, smoke, the default bench line, the launch list of the bench command
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-full}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err
  timeout 900 python bench.py --config C2 --sweep "" --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
  timeout 900 python bench.py --path dense --sweep "" --no-cpu-baseline --no-build > $OUT/bench_dense.json 2> $OUT/bench_dense.err
fi
if [ -z "$SKIP_NCU" ]; then
  timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 20 --warmup 3 --sweep "" --no-cpu-baseline > /dev/null 2>&1
  for k in ${FK:-estimate9 bucket_mark3 select_kernel merge_kernel qencode}; do
    timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/full_$k python tools/dec_bench.py C3 buckets=1 reps=2 > $OUT/ncu_$k.log 2>&1
  done
fi
ls -la $OUT
