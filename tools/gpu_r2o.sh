#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2o; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_gpu.py tests/test_bridges_dropin_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=5 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] (bridges)|parity" | tail -3; }
( run ETTG_HOOK_RUNS=1; run ETTG_HOOK_RUNS=0; run ETTG_HOOK_RUNS=1; run ETTG_HOOK_RUNS=0; run ETTG_HOOK_RUNS=1 GRAPH=C; run ETTG_HOOK_RUNS=0 GRAPH=C ) > $O/sweep.txt 2>&1
( for v in 1 0; do echo "== runs=$v"; ETTG_HOOK_RUNS=$v timeout 600 python tools/bridges_stress.py 2>&1 | tail -12; done ) > $O/stress.txt 2>&1
