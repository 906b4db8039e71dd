#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
s=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$? wall=$(( $(date +%s)-s ))" >> $O/rc.txt
