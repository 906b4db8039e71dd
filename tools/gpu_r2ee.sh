#!/bin/bash
# Compile-time hooking group (ETTG_CC_GROUP 4 / 8) vs the committed library; D and C.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ee}; mkdir -p $O
for rep in 1 2 3; do
  for v in old 4 8; do
    if [ $v = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; export ETTG_CC_GROUP=$v; fi
    echo "== $v rep $rep" >> $O/ab.txt
    ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C $v rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
    unset ETTG_CC_GROUP
  done
done
