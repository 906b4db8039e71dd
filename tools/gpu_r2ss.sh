#!/bin/bash
# low/high neighbour-lane run merge (ETTG_LH_MERGE) and the second-pass hash
# guard vs the committed library; config D / C traced; bridges tests with the merge on.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ss}; mkdir -p $O
for rep in 1 2 3; do
  for v in old 0 1; do
    if [ $v = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; export ETTG_LH_MERGE=$v; fi
    echo "== $v rep $rep" >> $O/ab.txt
    ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C $v rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
    unset ETTG_LH_MERGE
  done
done
unset AB_LIB
ETTG_LH_MERGE=1 timeout 900 python -m pytest tests -m gpu -q -x -k "bridge or tree or dropin" > $O/pytest_merge.log 2>&1; echo "pytest merge rc=$?" >> $O/rc.txt
