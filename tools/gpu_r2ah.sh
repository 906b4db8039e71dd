#!/bin/bash
# L1::no_allocate on the tour walk's successor loads (ETTG_LR_HINT=4) and the
# low/high filter reads (ETTG_LH_NA=1); config D and C traced.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ah}; mkdir -p $O
for rep in 1 2 3; do
  for v in "0 0" "4 0" "0 1" "4 1"; do
    set -- $v
    echo "== LR_HINT=$1 LH_NA=$2 rep $rep" >> $O/ab.txt
    ETTG_LR_HINT=$1 ETTG_LH_NA=$2 ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
done
for v in "0 0" "4 1"; do
  set -- $v
  echo "== C LR_HINT=$1 LH_NA=$2" >> $O/ab_C.txt
  GRAPH=C ETTG_LR_HINT=$1 ETTG_LH_NA=$2 ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
done
