#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2h; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu --durations=10 > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python tools/ab_bridges_e2e.py > $O/ab_br.txt 2>&1; echo "br rc=$?" >> $O/rc.txt
ETTG_TRACE=1 timeout 600 python tools/ab_lca_e2e.py 2>&1 | grep -v "^\[ettg trace\] \(build\|list\)" > $O/ab_lca.txt; echo "lca rc=$?" >> $O/rc.txt
s=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$? wall=$(( $(date +%s)-s ))" >> $O/rc.txt
