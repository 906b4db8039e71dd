#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python tools/ab_rawfrac.py > $O/rawfrac.txt 2>&1; echo "raw rc=$?" >> $O/rc.txt
timeout 900 bash tools/sweep_bridges.sh > $O/sweep.txt 2>&1; echo "sweep rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lr_walk0|k_lowhigh_edges|k_cc_hook" -c 4 -o $O/br_full env REPS=1 python tools/trace_bridges.py > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
