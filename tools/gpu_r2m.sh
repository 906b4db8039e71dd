#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2m; mkdir -p $O
timeout 900 python -m pytest tests/test_bridges_dropin_gpu.py tests/test_lca_gpu.py tests/test_multi_gpu.py tests/test_concurrency_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
ETTG_TRACE=1 timeout 900 python tools/ab_rawfrac.py > $O/rawfrac.txt 2>&1; echo "raw rc=$?" >> $O/rc.txt
