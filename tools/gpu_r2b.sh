#!/bin/bash
# iteration run: GPU tests (parity + buckets), decode micro-bench, launch list of the v7 kernels
cd "$(dirname "$0")/.."
OUT=gpurun_out/${R2OUT:-r2b}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_buckets.py -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
for spec in ${SPECS:-"C2" "C2:buckets=1" "C3" "C3:buckets=1"}; do
  timeout 300 python tools/dec_bench.py ${spec//:/ } >> $OUT/dec.jsonl 2>> $OUT/dec.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in ${LSPECS:-"C3:buckets=1" "C2"}; do
  tag=${spec//[:=]/_}
  timeout 600 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -c 40 --csv --log-file $OUT/launches_$tag.csv python tools/dec_bench.py ${spec//:/ } reps=2 > /dev/null 2>&1
  python tools/launches.py $OUT/launches_$tag.csv >> $OUT/launches.txt
done
tail -5 $OUT/pytest.log; cat $OUT/dec.jsonl; cat $OUT/launches.txt
