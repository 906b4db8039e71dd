#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus 2 --dist-backend gloo --same-device --steps 5 --no-bridges --no-cpu-baseline \
   --scaling-q 100000000 --scaling-steps 2 --e2e-steps 2 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo "2-rank rc=$?"; tail -c 600 gpurun_out/bench_2rank.json
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_lca_inlabel' -s 1 -c 2 \
   -o gpurun_out/prof_query -f python tools/prof_lca.py > gpurun_out/ncu_query.log 2>&1; echo "ncu rc=$?"
