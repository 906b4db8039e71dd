#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2oo}; mkdir -p $O
for rep in 1 2; do
  for v in -1 0; do
    echo "== LOCAL_HOOK=$v rep $rep" >> $O/ab.txt
    ETTG_LOCAL_HOOK=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
done
ETTG_LOCAL_HOOK=-1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:'k_local|k_cc_hook_list' --log-file $O/local.csv env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu.log 2>&1
