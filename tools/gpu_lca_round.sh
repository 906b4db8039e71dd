#!/bin/bash
# GPU tests, default bench, ncu launch list + full capture of the LCA query kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel' -s 1 -c 1 \
   -o gpurun_out/prof_query -f python tools/prof_lca.py > gpurun_out/ncu_query.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-scaling \
   --e2e-steps 1 --no-cpu-baseline --bridge-steps 1 > gpurun_out/ncu_launch_bench.json 2>&1; echo "launch list rc=$?"
