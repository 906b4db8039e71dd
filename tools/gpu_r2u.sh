#!/bin/bash
# ncu --set full of the config-D bridges kernels (second call), current code.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2u}; mkdir -p $O
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:'k_cc_hook|k_lowhigh_runs|k_lr_walk0|k_tree_rot|k_classify_tour|k_lh_block_ps|k_tv_keys|k_tree_close|k_compact_bits' \
   -s 10 -c 11 -o $O/prof_br -f env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_br2.log 2>&1; echo "br full rc=$?" >> $O/rc.txt
