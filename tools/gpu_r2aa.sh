#!/bin/bash
# Rotation variants (ETTG_ROT_V bit 0 prefetch, bit 1 close x4) + combined prefix/suffix array; D and C.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2aa}; mkdir -p $O
for rep in 1 2; do
  for v in 0 1 2 3; do
    echo "== ROT_V=$v rep $rep" >> $O/ab.txt
    ETTG_ROT_V=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
  echo "== C rep $rep" >> $O/ab_C.txt
  GRAPH=C ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
done
timeout 900 python -m pytest tests -m gpu -q -x -k "bridge or tree or dropin or cpp" > $O/pytest_br.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
