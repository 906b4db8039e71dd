#!/bin/bash
# Block-local hooking: config D traced (auto / off), config C, stress shapes, bridges tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2nn}; mkdir -p $O
for rep in 1 2; do
  for v in -1 0; do
    echo "== LOCAL_HOOK=$v rep $rep" >> $O/ab.txt
    ETTG_LOCAL_HOOK=$v ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/ab.txt
  done
done
GRAPH=C ETTG_TRACE=1 REPS=6 timeout 300 python tools/trace_bridges.py 2>&1 | tail -3 >> $O/ab_C.txt
timeout 600 python tools/bridges_stress.py > $O/stress.log 2>&1
ETTG_LOCAL_HOOK=1 timeout 600 python tools/bridges_stress.py > $O/stress_forced.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "bridge or tree or dropin" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
ETTG_LOCAL_HOOK=1 timeout 900 python -m pytest tests/test_bridges_gpu.py -m gpu -q -x > $O/pytest_forced.log 2>&1; echo "pytest forced rc=$?" >> $O/rc.txt
