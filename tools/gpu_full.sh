#!/bin/bash
# Round-end style GPU pass: tests, smoke, bench, reference arm, ncu launch list, trace.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-scaling \
   --e2e-steps 1 --no-cpu-baseline --bridge-steps 1 > gpurun_out/ncu_launch_bench.json 2>&1; echo "launch list rc=$?"
python tools/trace_bridges.py > gpurun_out/trace_br.log 2>&1; tail -3 gpurun_out/trace_br.log
