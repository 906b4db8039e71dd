#!/bin/bash
# ncu --set full captures of the top kernels after the round-1 tuning.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TREE=E timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel_split' -s 1 -c 1 \
   -o gpurun_out/prof_split -f python tools/prof_lca.py > gpurun_out/ncu_split.log 2>&1; echo "split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'k_cc_hook|k_lowhigh_edges|k_lr_walk0|k_classify|k_scan_dlb|k_compact_u8|k_tree_rot' \
   -c 40 -o gpurun_out/prof_br -f env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > gpurun_out/ncu_br.log 2>&1; echo "bridges rc=$?"
