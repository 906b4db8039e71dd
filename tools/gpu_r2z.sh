#!/bin/bash
# Rotation prefetch / close unroll: traced config D + C, bridges GPU tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2z}; mkdir -p $O
for rep in 1 2 3; do
  echo "== new rep $rep" >> $O/ab.txt
  ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  echo "== C new rep $rep" >> $O/ab_C.txt
  GRAPH=C ETTG_TRACE=1 REPS=8 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab_C.txt
done
timeout 900 python -m pytest tests -m gpu -q -x -k "bridge or tree or dropin or cpp" > $O/pytest_br.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
