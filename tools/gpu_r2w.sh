#!/bin/bash
# list-ranking level means (ETTG_LR_L0 / ETTG_LR_L) and hooking prefetch (ETTG_HOOK_PF) A/B on config D.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2w}; mkdir -p $O
for rep in 1 2; do
  for v in "16 16 0" "16 4 0" "16 8 0" "8 4 0" "8 8 0" "16 16 1" "16 16 2" "16 16 3"; do
    set -- $v
    echo "== LR_L0=$1 LR_L=$2 HOOK_PF=$3 rep $rep" >> $O/ab.txt
    ETTG_LR_L0=$1 ETTG_LR_L=$2 ETTG_HOOK_PF=$3 ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
done
