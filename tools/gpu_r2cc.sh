#!/bin/bash
# A/B vs the committed library (tools/_old/libettg_head.so): config D and C traced.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2cc}; mkdir -p $O
for rep in 1 2 3; do
  for lib in old new; do
    if [ $lib = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; fi
    echo "== $lib rep $rep" >> $O/ab.txt
    ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C $lib rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
  done
done
unset AB_LIB
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$TESTS" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt; fi
