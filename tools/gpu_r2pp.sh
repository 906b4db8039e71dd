#!/bin/bash
# Streaming-store widening / mask expansion vs the committed library: pageable
# paths (tools/ab_pageable.py) and the bench's pinned e2e lines; GPU tests that
# cover the host copies.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2pp}; mkdir -p $O
for rep in 1 2 3; do
  for lib in old new; do
    if [ $lib = old ]; then export AB_LIB=$PWD/tools/_old/libettg_head.so; else unset AB_LIB; fi
    echo "== $lib rep $rep" >> $O/pageable.txt
    timeout 600 python tools/ab_pageable.py >> $O/pageable.txt 2>&1
  done
done
unset AB_LIB
timeout 900 python -m pytest tests -m gpu -q -x -k "query or batch or bridge or stats or export or parse or adjacency" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
