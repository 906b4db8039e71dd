#!/bin/bash
# Env-knob sweep of TV bridges on config D (device-resident edges), ETTG_TRACE
# phase lines + the PhaseTimes totals of the last 2 of 4 calls (dev aid).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
run() { echo "== $*"; env "$@" ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | grep -E "^bridges|\[ettg trace\] (bridges|list_rank)" | tail -6; }
run X=base
run ETTG_LR_L0=32
run ETTG_LR_L0=8
run ETTG_CC_SAMPLE=8
run ETTG_CC_SAMPLE=2
run ETTG_LH_CHECK=0
run ETTG_LR_WYLLIE=0
