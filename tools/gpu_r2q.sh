#!/bin/bash
# L2 eviction-hint A/B on the query kernels (ETTG_L2HINT 0/1/2, alternating),
# then the per-kernel DRAM of one config-D bridges call and its phase trace.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/${TAG:-r2q}; mkdir -p $O
for rep in 1 2; do
  for h in 0 1 2; do
    ETTG_L2HINT=$h AB_ONLY=B_path,E_rand,g8,g64 timeout 600 python tools/ab_lca.py auto >> $O/l2hint_$h.txt 2>&1
  done
done
if [ -z "$NO_BR" ]; then
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --csv --log-file $O/br_dram.csv \
   env ETTG_TRACE=0 REPS=2 python tools/trace_bridges.py > $O/ncu_br.log 2>&1; echo "br dram rc=$?" >> $O/rc.txt
ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py > $O/trace_br.log 2>&1
fi
# streamed-edge cache policy A/B (ETTG_BR_CS bit 0 hooking, bit 1 low/high)
for rep in 1 2; do
  for c in 0 1 2 3; do
    echo "== BR_CS=$c rep $rep" >> $O/brcs.txt
    ETTG_BR_CS=$c ETTG_TRACE=1 REPS=4 timeout 300 python tools/trace_bridges.py 2>&1 | tail -4 >> $O/brcs.txt
  done
done
