#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_gpu.py tests/test_primitives_gpu.py tests/test_lca_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] (bridges|list_rank)|parity" | tail -4; }
( run ETTG_LR_SORTED=1; run ETTG_LR_SORTED=0; run ETTG_LR_SORTED=1 GRAPH=C; run ETTG_LR_SORTED=0 GRAPH=C ) > $O/sweep.txt 2>&1
( for v in 1 0; do echo "== sorted=$v"; ETTG_LR_SORTED=$v ETTG_TRACE=1 timeout 300 python tools/trace_build.py 2>&1 | grep -E "lca_build|list_rank" | tail -4; done ) > $O/build.txt 2>&1
