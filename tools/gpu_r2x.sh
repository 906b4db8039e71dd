#!/bin/bash
# list-ranking level means (ETTG_LR_L0 / ETTG_LR_L) on config D bridges and the 16M LCA builds;
# low/high prefetch (ETTG_LH_MINB=14).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2x}; mkdir -p $O
for rep in 1 2; do
  for v in "16 16 5" "8 4 5" "8 2 5" "4 4 5" "4 2 5" "8 4 14"; do
    set -- $v
    echo "== LR_L0=$1 LR_L=$2 LH_MINB=$3 rep $rep" >> $O/ab.txt
    ETTG_LR_L0=$1 ETTG_LR_L=$2 ETTG_LH_MINB=$3 ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== LR_L0=$1 LR_L=$2 rep $rep" >> $O/build.txt
    ETTG_LR_L0=$1 ETTG_LR_L=$2 timeout 300 python tools/trace_build.py 2>&1 | grep -v "^\[ettg trace\] lca_build\|^$" | tail -12 >> $O/build.txt
  done
done
