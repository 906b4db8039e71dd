#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2n2; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_gpu.py tests/test_bridges_dropin_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=5 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] (bridges)|parity" | tail -3; }
( run ETTG_LH_RUNS=1; run ETTG_LH_RUNS=0; run ETTG_LH_RUNS=1; run ETTG_LH_RUNS=0; run ETTG_LH_RUNS=1 GRAPH=C; run ETTG_LH_RUNS=0 GRAPH=C ) > $O/sweep.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:'k_lowhigh' -s 1 -c 1 -o $O/prof -f env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu.log 2>&1
