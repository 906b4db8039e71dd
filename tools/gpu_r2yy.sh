#!/bin/bash
# Predicated low/high (ETTG_LH_PRED) A/B on config D; bridges tests with it on.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2yy}; mkdir -p $O
for rep in 1 2 3; do
  for v in 0 1; do
    echo "== LH_PRED=$v rep $rep" >> $O/ab.txt
    ETTG_LH_PRED=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
done
ETTG_LH_PRED=1 timeout 600 python tools/bridges_stress.py > $O/stress.log 2>&1
