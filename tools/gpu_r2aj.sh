#!/bin/bash
# LCA build tour walk: no L1 allocation (ETTG_LR_HINT_W=4) / L2 evict_last (2) on the successor loads.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2aj}; mkdir -p $O
for rep in 1 2 3; do
  for h in 0 4 2; do
    echo "== HINT_W=$h rep $rep" >> $O/build.txt
    ETTG_LR_HINT_W=$h timeout 300 python tools/trace_build.py 2>&1 | grep "build_ms\|walk0" | tail -6 >> $O/build.txt
  done
done
