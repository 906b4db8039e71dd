#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_gpu.py tests/test_bridges_dropin_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] bridges|parity" | tail -3; }
( run X=D; run GRAPH=C ) > $O/sweep.txt 2>&1
timeout 600 python tools/ab_bridges_e2e_trace.py > $O/e2e.txt 2>&1
