#!/bin/bash
# Round-2 full pass: gpu tests, smoke, bench (ours + reference arm), ncu launch
# list of the bench command, --set full of the top kernels, per-kernel DRAM of
# one config-D bridges call, bridges phase trace.  Output: gpurun_out/$TAG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2full}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
if [ -z "$NO_BENCH" ]; then
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/rc.txt
fi
if [ -z "$NO_PROF" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
   --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-scaling \
   --e2e-steps 1 --no-cpu-baseline --bridge-steps 1 > $O/ncu_launch_bench.json 2>&1; echo "launch rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel' -s 1 -c 1 \
   -o $O/prof_query -f python tools/prof_lca.py > $O/ncu_query.log 2>&1; echo "ncu B rc=$?" >> $O/rc.txt
TREE=E timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel' -s 1 -c 1 \
   -o $O/prof_split6 -f python tools/prof_lca.py > $O/ncu_split.log 2>&1; echo "ncu E rc=$?" >> $O/rc.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file $O/br_dram.csv \
   env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_br.log 2>&1; echo "br dram rc=$?" >> $O/rc.txt
timeout 1200 ncu --set full --clock-control none --import-source on \
   -k regex:'k_cc_hook|k_lowhigh|k_lr_walk0|k_tree_rot|k_classify_tour|k_lh_block_ps|k_tv_keys|k_compact_bits|k_tree_close' \
   -s 10 -c 11 -o $O/prof_br -f env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_br2.log 2>&1; echo "br full rc=$?" >> $O/rc.txt
ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py > $O/trace_br.log 2>&1
fi
du -sh $O
