#!/bin/bash
# Index gathers: evict_last (ETTG_L2HINT=1), + L1::no_allocate on the compact words (3),
# + L1::no_allocate on the split6 sectors too (4).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ag}; mkdir -p $O
for rep in 1 2 3; do
  for h in 1 3 4; do
    ETTG_L2HINT=$h AB_ONLY=B_path,E_rand,g64,path_4M,rand_4M timeout 600 python tools/ab_lca.py auto >> $O/l2hint_$h.txt 2>&1
  done
done
