#!/bin/bash
# Query launch shape re-check with the no-allocate gathers: grid CTAs/SM and pair-prefetch mode.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2ak}; mkdir -p $O
for rep in 1 2; do
  for g in 8 16 32 64 128; do
    for pf in 1 2; do
      echo "== QGRID=$g QPF=$pf rep $rep" >> $O/ab.txt
      ETTG_QGRID=$g ETTG_QPF=$pf AB_ONLY=B_path,E_rand timeout 600 python tools/ab_lca.py auto >> $O/ab.txt 2>&1
    done
  done
done
