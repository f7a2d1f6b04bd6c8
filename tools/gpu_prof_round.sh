#!/bin/bash
# round evidence: GPU tests, bench (with context sweep), ncu launch list + --set full, summaries
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
TAG=${TAG:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --sweep "C2:4096,C2:16384,C2:65536,C2:131072,C3,C2b:16384,C2b:131072,C3b" > $OUT/bench.log 2>&1
echo "bench exit $?" >> $OUT/bench.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 64 --warmup 3 --no-cpu-baseline --replicas 2 --e2e-steps 8 --sweep "" > $OUT/ncu_launches.log 2>&1
echo "ncu1 exit $?" >> $OUT/ncu_launches.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"decode5_kernel|qencode_kernel|hash_gemm_kernel" -s 2 -c 5 \
   -o $OUT/full python bench.py --steps 16 --warmup 3 --no-cpu-baseline --replicas 2 --e2e-steps 4 --sweep "" > $OUT/ncu_full.log 2>&1
echo "ncu2 exit $?" >> $OUT/ncu_full.log
timeout 300 python tools/timeline.py C2 > $OUT/timeline_c2.log 2>&1
