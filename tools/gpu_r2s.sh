#!/bin/bash
# Tree bits: bridges GPU tests, then A/B vs the previous library (tools/_old/libettg_head.so).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2s}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "bridge or bfs or ck or hybrid or tree or dropin or cpp or parse" > $O/pytest_br.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for rep in 1 2; do
  for lib in old new; do
    echo "== $lib rep $rep" >> $O/ab.txt
    if [ $lib = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; fi
    ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -3 >> $O/ab.txt
    GRAPH=C ETTG_TRACE=1 REPS=6 timeout 300 python tools/trace_bridges.py 2>&1 | tail -2 >> $O/ab_C.txt
  done
done
unset AB_LIB
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file $O/br_dram.csv \
   env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_br.log 2>&1; echo "br dram rc=$?" >> $O/rc.txt
