#!/bin/bash
# Speculative next-successor load in the bridges tour walk (ETTG_LR_SPEC).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2xx}; mkdir -p $O
for rep in 1 2 3; do
  for v in 0 1; do
    echo "== LR_SPEC=$v rep $rep" >> $O/ab.txt
    ETTG_LR_SPEC=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
    echo "== C LR_SPEC=$v rep $rep" >> $O/ab_C.txt
    GRAPH=C ETTG_LR_SPEC=$v ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
  done
done
ETTG_LR_SPEC=1 timeout 900 python -m pytest tests -m gpu -q -x -k "bridge or tree or dropin or list_rank" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
ETTG_LR_SPEC=1 timeout 600 python tools/bridges_stress.py > $O/stress.log 2>&1
