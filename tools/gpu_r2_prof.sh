#!/bin/bash
# Round-2 profile pass: ncu launch list of the bench command, --set full of
# the top kernels, DRAM bytes per kernel of one config-D bridges call, and the
# bridges phase trace.  Output under gpurun_out/$TAG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2p}; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
   --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-scaling \
   --e2e-steps 1 --no-cpu-baseline --bridge-steps 1 > $O/ncu_launch_bench.json 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel' -s 1 -c 1 \
   -o $O/prof_query -f python tools/prof_lca.py > $O/ncu_query.log 2>&1; echo "compact rc=$?"
TREE=E timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel' -s 1 -c 1 \
   -o $O/prof_split6 -f python tools/prof_lca.py > $O/ncu_split.log 2>&1; echo "split6 rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file $O/br_dram.csv \
   env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_br.log 2>&1; echo "bridges dram rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
   -k regex:'k_cc_hook|k_lowhigh_edges|k_lr_walk0|k_tree_rot|k_classify_tour|k_lh_block_ps|k_tv_keys' \
   -s 8 -c 8 -o $O/prof_br -f env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_br2.log 2>&1; echo "bridges full rc=$?"
ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py > $O/trace_br.log 2>&1; echo "trace rc=$?"
du -sh $O
