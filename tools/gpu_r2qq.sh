#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2qq}; mkdir -p $O
for rep in 1 2 3 4; do
  for lib in old new; do
    if [ $lib = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; fi
    echo "== $lib rep $rep" >> $O/nt.txt
    timeout 600 python tools/ab_e2e_nt.py >> $O/nt.txt 2>&1
  done
done
