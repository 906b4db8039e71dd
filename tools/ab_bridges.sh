#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export ETTG_TRACE=1
REPS=4 python tools/prof_bridges.py 2>&1 | grep -E "trace\] bridges|parity" | tail -3
