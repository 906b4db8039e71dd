#!/bin/bash
# Host-side e2e characterisation: host topology, host narrowing rate, staged
# upload pipeline, PCIe duplex, and the raw-fraction sweep with traces.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2e}; mkdir -p $O
bash tools/probe_box.sh > $O/probe.txt 2>&1
numactl -H >> $O/probe.txt 2>&1; cat /proc/meminfo | head -5 >> $O/probe.txt
timeout 300 tools/_bin/host_narrow_micro > $O/host_narrow.txt 2>&1
timeout 300 tools/_bin/pcie_micro > $O/pcie.txt 2>&1
timeout 300 tools/_bin/stage_micro > $O/stage.txt 2>&1
ETTG_TRACE=1 timeout 900 python tools/ab_rawfrac.py > $O/rawfrac.txt 2>&1; echo "raw rc=$?"
