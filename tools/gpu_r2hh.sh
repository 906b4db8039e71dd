#!/bin/bash
# Sampled-pass thread-to-edge mapping (ETTG_HOOK_ADJ) on config D and C.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2hh}; mkdir -p $O
for rep in 1 2; do
  for v in 0 1 2 3; do
    echo "== HOOK_ADJ=$v rep $rep" >> $O/ab.txt
    ETTG_HOOK_ADJ=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C HOOK_ADJ=$v rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_HOOK_ADJ=$v ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
  done
done
