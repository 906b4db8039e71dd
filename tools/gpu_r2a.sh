#!/bin/bash
# round-2 first GPU pass: full-scale parity tests, small + full bench, reference arm
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2a; mkdir -p $O
timeout 300 python bench.py --n 1000000 --q 1000000 --scaling-q 10000000 --road-side 1000 --road-pendant 1000 --e-sample 1000000 --steps 3 --warmup 3 > $O/bench_small.json 2> $O/bench_small.err; echo "small rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_fullscale_gpu.py -x -q -m gpu --durations=0 > $O/fullscale.txt 2>&1; echo "full rc=$?" >> $O/rc.txt
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?" >> $O/rc.txt
/usr/bin/time -v timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
