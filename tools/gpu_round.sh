#!/bin/bash
# One GPU session: small bench smoke, full bench, ncu launch list, ncu full captures.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 600 python bench.py --n 100000 --q 100000 --scaling-q 1000000 --road-side 200 \
    --road-pendant 500 --cpu-road-side 100 --steps 10 > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err
echo "small rc=$?"
if [ "${FULL:-1}" = "1" ]; then
  timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "full rc=$?"
  timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  echo "ref rc=$?"
fi
if [ "${PROFILE:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-scaling \
      --e2e-steps 1 --no-cpu-baseline --bridge-steps 1 > gpurun_out/ncu_launch_bench.json 2>&1
  echo "launch list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:'k_lca_inlabel|k_cc_hook|k_lr_walk0|k_lowhigh_edges|k_classify|k_tree_succ|k_rs_scatter' \
      -c 12 -o gpurun_out/prof_full -f python bench.py --steps 2 --warmup 1 --no-scaling \
      --e2e-steps 1 --no-cpu-baseline --bridge-steps 1 > gpurun_out/ncu_full.log 2>&1
  echo "full capture rc=$?"
fi
