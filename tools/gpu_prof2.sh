#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
ETTG_TRACE=1 python tools/trace_run.py 2>&1 | grep -v -E "Exception|Traceback|File|TypeError" > gpurun_out/trace2.log
python -m pytest tests -m gpu -q -x > gpurun_out/pytest4.log 2>&1; tail -3 gpurun_out/pytest4.log
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'k_cc_hook|k_lowhigh_edges|k_classify|k_tree_rot|k_tree_succ|k_lr_walk0|k_compact_u8|k_tour_flags' \
   -s 8 -c 9 -o gpurun_out/prof_bridges -f python tools/prof_bridges.py > gpurun_out/ncu_bridges.log 2>&1
echo "ncu bridges rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel|k_asc_level|k_lr_walk0|k_rs_scatter' \
   -c 8 -o gpurun_out/prof_lca -f python tools/prof_lca.py > gpurun_out/ncu_lca.log 2>&1
echo "ncu lca rc=$?"
cat gpurun_out/trace2.log
