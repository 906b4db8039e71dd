#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fopenmp tools/stage_micro.cu -o /tmp/stage_micro && /tmp/stage_micro > $O/stage_micro.txt 2>&1
ETTG_TRACE=1 timeout 600 python tools/ab_lca_e2e.py > $O/ab_lca.txt 2>&1; echo "lca rc=$?" >> $O/rc.txt
