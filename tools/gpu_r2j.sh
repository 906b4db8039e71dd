#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2j; mkdir -p $O
timeout 900 python -m pytest tests/test_primitives_gpu.py tests/test_bridges_gpu.py tests/test_lca_gpu.py tests/test_bridges_dropin_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] (bridges|list_rank)" | tail -4; }
( run X=base; run ETTG_LR_L0=32; run ETTG_LR_L0=64; run GRAPH=C; run GRAPH=C ETTG_LR_L0=32 ) > $O/sweep.txt 2>&1
timeout 600 python tools/trace_build.py > $O/build.txt 2>&1; echo "build rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lr_walk0" -c 1 -o $O/walk0 env REPS=1 python tools/trace_bridges.py > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
