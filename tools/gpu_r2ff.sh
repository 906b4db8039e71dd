#!/bin/bash
# Per-kernel durations of the hooking passes, committed vs working library.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ff}; mkdir -p $O
for lib in old new; do
  if [ $lib = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__registers_per_thread,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv -k regex:'k_cc_' --log-file $O/hook_$lib.csv env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_$lib.log 2>&1
done
