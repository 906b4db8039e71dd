#!/bin/bash
# Sampled pass with priority linking (ETTG_HOOK_PRIO0) on config D and C.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2af}; mkdir -p $O
for rep in 1 2 3; do
  for v in 0 1; do
    echo "== PRIO0=$v rep $rep" >> $O/ab.txt
    ETTG_HOOK_PRIO0=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C PRIO0=$v rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_HOOK_PRIO0=$v ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
  done
done
ETTG_HOOK_PRIO0=1 timeout 600 python tools/bridges_stress.py > $O/stress.log 2>&1
