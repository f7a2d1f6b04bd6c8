#!/bin/bash
# GPU tests + timeline + bench (no ncu)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/timeline.py C2 > gpurun_out/timeline_c2.log 2>&1
timeout 600 python bench.py --steps 2000 --warmup 64 --cpu-seconds 3 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
