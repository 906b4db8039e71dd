#!/bin/bash
# LCA build list-ranking level means (ETTG_LR_L0 / ETTG_LR_L) on the 16M path and random trees.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ab}; mkdir -p $O
for rep in 1 2; do
  for v in "16 16" "32 8" "32 16" "64 8" "32 4"; do
    set -- $v
    echo "== LR_L0=$1 LR_L=$2 rep $rep" >> $O/build.txt
    ETTG_LR_L0=$1 ETTG_LR_L=$2 timeout 300 python tools/trace_build.py 2>&1 | grep "build_ms" >> $O/build.txt
  done
done
