#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2g; mkdir -p $O
for f in "-O3" "-O3 -march=x86-64-v3" "-O3 -march=x86-64-v4" "-O3 -march=native"; do
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fopenmp -Xcompiler "$f" tools/stage_micro.cu -o /tmp/sm && echo "== $f" >> $O/stage.txt && /tmp/sm 2>&1 | grep -E "plain|16 MB|8 MB x 3" >> $O/stage.txt
done
