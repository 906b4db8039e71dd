#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b; mkdir -p $O
g++ -O3 -march=native -fopenmp tools/host_narrow_micro.cpp -o /tmp/hn && /tmp/hn > $O/host_narrow.txt 2>&1
s=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$? wall=$(( $(date +%s)-s ))" >> $O/rc.txt
