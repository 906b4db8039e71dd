#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2m2; mkdir -p $O
ETTG_QPF=2 timeout 600 python -m pytest tests/test_lca_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 1 2; do
for v in "ETTG_QPF=1" "ETTG_QPF=2" "ETTG_QPF=2 ETTG_QGRID=8" "ETTG_QPF=2 ETTG_QGRID=16"; do
  echo "== $v" >> $O/ab.txt
  env $v AB_ONLY=B_path,path_1M,path_4M timeout 300 python tools/ab_lca.py auto >> $O/ab.txt 2>&1
done; done
