#!/bin/bash
# Hooking rounds A/B on config D and C (ETTG_CC_ROUNDS / ETTG_CC_SAMPLE), traced.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2r}; mkdir -p $O
for rep in 1 2; do
  for v in "1 4" "2 8" "2 6" "3 12" "2 4"; do
    set -- $v
    echo "== rounds=$1 sample=$2 rep $rep" >> $O/rounds.txt
    ETTG_CC_ROUNDS=$1 ETTG_CC_SAMPLE=$2 ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -3 >> $O/rounds.txt
    echo "== C rounds=$1 sample=$2 rep $rep" >> $O/rounds_C.txt
    GRAPH=C ETTG_CC_ROUNDS=$1 ETTG_CC_SAMPLE=$2 ETTG_TRACE=1 REPS=6 timeout 300 python tools/trace_bridges.py 2>&1 | tail -3 >> $O/rounds_C.txt
  done
done
