#!/bin/bash
# Level-0 walk cache hints A/B on config D (ETTG_LR_HINT 0..3).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2t}; mkdir -p $O
for rep in 1 2; do
  for h in 0 1 2 3; do
    echo "== LR_HINT=$h rep $rep" >> $O/lrhint.txt
    ETTG_LR_HINT=$h ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/lrhint.txt
  done
done
