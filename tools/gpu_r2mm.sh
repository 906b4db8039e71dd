#!/bin/bash
# Where the bench's config-D number differs from the standalone trace.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2mm}; mkdir -p $O
timeout 900 python bench.py --no-scaling --no-cpu-baseline --steps 20 --e2e-steps 1 > $O/b_noscale.json 2> $O/b_noscale.err
ETTG_TRACE=1 timeout 900 python bench.py --no-scaling --no-cpu-baseline --steps 20 --e2e-steps 1 > $O/b_noscale_tr.json 2> $O/b_noscale_tr.err
timeout 900 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 1 > $O/b_full.json 2> $O/b_full.err
ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py > $O/trace.log 2>&1
