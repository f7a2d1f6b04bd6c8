#!/bin/bash
# A/B of decode-kernel variants (debug knob kernel=5,15,25,35): parity tests of the decode, timeline, micro-bench
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
OUT=gpurun_out/${TAG:-ab}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 300 > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
for kv in ${KVERS:-5 15 35}; do
  echo "== kernel $kv" >> $OUT/dec.log
  timeout 120 python tools/dec_bench.py C2 kernel=$kv >> $OUT/dec.log 2>&1
  timeout 300 python tools/dec_bench.py C2 n=131072 reps=2 kernel=$kv >> $OUT/dec.log 2>&1
  timeout 600 python tools/dec_bench.py C3 reps=2 kernel=$kv >> $OUT/dec.log 2>&1
done
timeout 120 python tools/timeline.py C2 > $OUT/timeline_c2.log 2>&1
