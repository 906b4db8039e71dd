#!/bin/bash
# ncu --set full captures of the top kernels (one launch each) and the DRAM
# bytes of every kernel of one bridges call (3 metrics, CSV).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel' -s 1 -c 1 \
   -o gpurun_out/prof_query -f python tools/prof_lca.py > gpurun_out/ncu_query.log 2>&1; echo "compact rc=$?"
TREE=E timeout 600 ncu --set full --clock-control none -k regex:'k_lca_inlabel' -s 1 -c 1 \
   -o gpurun_out/prof_split6 -f python tools/prof_lca.py > gpurun_out/ncu_split.log 2>&1; echo "split6 rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/br_dram.csv \
   env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > gpurun_out/ncu_br.log 2>&1; echo "bridges dram rc=$?"
timeout 1200 ncu --set full --clock-control none \
   -k regex:'k_cc_hook|k_lowhigh_edges|k_lr_walk0|k_tree_rot|k_classify_tour|k_lh_block_ps' \
   -s 7 -c 7 -o gpurun_out/prof_br -f env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > gpurun_out/ncu_br2.log 2>&1; echo "bridges full rc=$?"
du -sh gpurun_out
