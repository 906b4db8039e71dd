#!/bin/bash
# split6 query grid (ETTG_QGRID) on the E shape (64M queries) and the 1G-query E stream.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2al}; mkdir -p $O
for rep in 1 2; do
  for g in 64 128 256 512; do
    echo "== QGRID=$g rep $rep" >> $O/ab.txt
    ETTG_QGRID=$g AB_ONLY=E_rand,g64,rand_4M timeout 600 python tools/ab_lca.py auto >> $O/ab.txt 2>&1
  done
done
for g in 64 128 256; do
  echo "== bench E QGRID=$g" >> $O/benchE.txt
  ETTG_QGRID=$g timeout 900 python bench.py --no-cpu-baseline --no-bridges --steps 5 --e2e-steps 1 --scaling-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']/1e9, d['scaling_config_E']['value']/1e9)" >> $O/benchE.txt
done
