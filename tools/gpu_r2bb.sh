#!/bin/bash
# Sampled-pass find shortcut threshold (ETTG_HOOK_SC) on config D and C.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2bb}; mkdir -p $O
for rep in 1 2; do
  for v in 8 2 4 16 99; do
    echo "== HOOK_SC=$v rep $rep" >> $O/ab.txt
    ETTG_HOOK_SC=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C HOOK_SC=$v rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_HOOK_SC=$v ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
  done
done
