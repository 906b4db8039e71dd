#!/bin/bash
# wide9 gathers without L1 allocation (ETTG_L2HINT=4 vs 1) on the middle-depth trees.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ai}; mkdir -p $O
for rep in 1 2 3; do
  for h in 1 4; do
    ETTG_L2HINT=$h AB_ONLY=g4,g8,g16,g2 timeout 600 python tools/ab_lca.py auto >> $O/l2hint_$h.txt 2>&1
  done
done
