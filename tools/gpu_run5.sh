#!/bin/bash
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 300 python tools/timeline.py C2 > gpurun_out/timeline_c2.log 2>&1
