#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2e; mkdir -p $O
timeout 600 python tools/ab_lca_e2e.py > $O/ab_lca.txt 2>&1; echo "lca rc=$?" >> $O/rc.txt
timeout 900 python tools/ab_bridges_e2e.py > $O/ab_br.txt 2>&1; echo "br rc=$?" >> $O/rc.txt
timeout 600 bash tools/gpu_br_dram.sh > $O/dram.txt 2>&1; cp gpurun_out/br_dram.csv $O/ 2>/dev/null; echo "dram rc=$?" >> $O/rc.txt
