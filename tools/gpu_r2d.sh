#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu --durations=20 > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
s=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$? wall=$(( $(date +%s)-s ))" >> $O/rc.txt
