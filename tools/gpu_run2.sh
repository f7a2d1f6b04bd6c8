#!/bin/bash
# GPU session: tests, bench, ncu launch list + full profile of the decode kernels
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -rA > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2000 --warmup 64 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 64 --warmup 3 --no-cpu-baseline --replicas 2 --e2e-steps 8 > gpurun_out/ncu_bench.log 2>&1
echo "ncu1 exit $?" >> gpurun_out/ncu_bench.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"decode_kernel|qencode_kernel" -s 20 -c 4 \
   -o gpurun_out/decode_full python bench.py --steps 64 --warmup 3 --no-cpu-baseline --replicas 2 --e2e-steps 8 > gpurun_out/ncu_full.log 2>&1
echo "ncu2 exit $?" >> gpurun_out/ncu_full.log
