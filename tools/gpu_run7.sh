#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
./tools/micro/latency > gpurun_out/latency.log 2>&1
timeout 300 python tools/build_once.py C2 > gpurun_out/build_c2.log 2>&1
timeout 300 python tools/build_once.py C3 > gpurun_out/build_c3.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"hash_gemm_kernel|key_stats|prep_x|fixup" -c 4 \
   -o gpurun_out/build_full python tools/build_once.py C2 > gpurun_out/ncu_build.log 2>&1
