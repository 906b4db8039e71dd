#!/bin/bash
# low/high occupancy (ETTG_LH_MINB) and level-0 sublist length (ETTG_LR_L0) A/B on config D.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2v}; mkdir -p $O
for rep in 1 2; do
  for v in "4 16" "5 16" "6 16" "4 8" "4 32"; do
    set -- $v
    echo "== LH_MINB=$1 LR_L0=$2 rep $rep" >> $O/ab.txt
    ETTG_LH_MINB=$1 ETTG_LR_L0=$2 ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
done
