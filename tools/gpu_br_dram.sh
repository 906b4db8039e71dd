#!/bin/bash
# DRAM bytes of every kernel of one tv_bridges call on config D (3 metrics, CSV).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file gpurun_out/br_dram.csv \
   env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > gpurun_out/ncu_br.log 2>&1; echo "bridges dram rc=$?"
