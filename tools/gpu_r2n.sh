#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2n; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_gpu.py tests/test_bridges_dropin_gpu.py tests/test_cpp_shim.py tests/test_primitives_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] (bridges|list_rank)|parity" | tail -4; }
( run X=D; run GRAPH=C; run ETTG_LR_NARROW=0 ) > $O/sweep.txt 2>&1
