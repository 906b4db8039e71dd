#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2k; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_gpu.py tests/test_bridges_dropin_gpu.py tests/test_cpp_shim.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] bridges|parity" | tail -3; }
( run ETTG_LH_AGG=1; run ETTG_LH_AGG=0; run GRAPH=C ETTG_LH_AGG=1; run GRAPH=C ETTG_LH_AGG=0 ) > $O/sweep.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lowhigh_edges" -c 1 -o $O/lh env REPS=1 python tools/trace_bridges.py > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
