#!/bin/bash
# ncu --set full (source-level) of the two hooking passes, config D.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2uu}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cc_hook' -s 2 -c 2 \
   -o $O/prof_hook -f env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu.log 2>&1; echo "rc=$?" >> $O/rc.txt
