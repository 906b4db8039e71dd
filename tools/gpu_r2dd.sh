#!/bin/bash
# Sampled-pass group size (ETTG_CC_GROUP) x sample rate on config D and C.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2dd}; mkdir -p $O
for rep in 1 2; do
  for v in "4 4" "8 4" "16 4" "32 4" "8 3" "16 3"; do
    set -- $v
    echo "== GROUP=$1 SAMPLE=$2 rep $rep" >> $O/ab.txt
    ETTG_CC_GROUP=$1 ETTG_CC_SAMPLE=$2 ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C GROUP=$1 SAMPLE=$2 rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_CC_GROUP=$1 ETTG_CC_SAMPLE=$2 ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
  done
done
