#!/bin/bash
# tests + bench + ncu evidence (launch list + --set full of the decode, encode and hash kernels)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2000 --warmup 64 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 64 --warmup 3 --no-cpu-baseline --replicas 2 --e2e-steps 8 > gpurun_out/ncu_bench.log 2>&1
echo "ncu1 exit $?" >> gpurun_out/ncu_bench.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"decode_kernel|qencode_kernel|hash_gemm_kernel" -s 2 -c 5 \
   -o gpurun_out/full python bench.py --steps 16 --warmup 3 --no-cpu-baseline --replicas 2 --e2e-steps 4 > gpurun_out/ncu_full.log 2>&1
echo "ncu2 exit $?" >> gpurun_out/ncu_full.log
timeout 300 python tools/timeline.py C2 > gpurun_out/timeline_c2.log 2>&1
