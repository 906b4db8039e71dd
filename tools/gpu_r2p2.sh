#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2q; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_gpu.py tests/test_parse_gpu.py tests/test_bridges_dropin_gpu.py tests/test_primitives_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=5 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] (bridges)|parity" | tail -3; }
( run ETTG_COMPACT_2PASS=1; run ETTG_COMPACT_2PASS=0; run ETTG_COMPACT_2PASS=1; run ETTG_COMPACT_2PASS=0; run ETTG_COMPACT_2PASS=1 GRAPH=C; run ETTG_COMPACT_2PASS=0 GRAPH=C ) > $O/sweep.txt 2>&1
