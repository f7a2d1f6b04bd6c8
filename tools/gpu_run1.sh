#!/bin/bash
# first GPU session: tests, smoke, short bench
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -rA > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 2000 --warmup 64 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
