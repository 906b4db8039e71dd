#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ll}; mkdir -p $O
for rep in 1 2; do
  ETTG_TRACE=0 timeout 300 python tools/bridges_timing_modes.py >> $O/modes.txt 2>&1
  ETTG_TRACE=1 timeout 300 python tools/bridges_timing_modes.py 2>/dev/null >> $O/modes.txt
  AB_LIB=x true
done
for rep in 1 2 3; do
  for lib in old new; do
    if [ $lib = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; fi
    echo "== $lib rep $rep" >> $O/ab.txt
    ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
done
