#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2g; mkdir -p $O
timeout 600 python -m pytest tests/test_lca_gpu.py tests/test_multi_gpu.py tests/test_concurrency_gpu.py tests/test_bridges_dropin_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python tools/ab_pipe.py > $O/ab.txt 2>&1; echo "ab rc=$?" >> $O/rc.txt
ETTG_TRACE=1 VARIANTS="ETTG_PIPE=1" SKIP_BR=1 timeout 300 python tools/ab_pipe.py > $O/trace.txt 2>&1
