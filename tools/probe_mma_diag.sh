#!/bin/bash
# Family / width / diagnostic-switch sweep of the mma.sync GEMM on the gate-up shape with the diag library.
FMS=${FMS:-"0:8 2:8 2:16"}
DBGS=${DBGS:-"0 2"}
for fm in $FMS; do f=${fm%%:*}; m=${fm##*:}
for dbg in $DBGS; do
  W4A16_LIB=diag W4A16_MMA_DEBUG=$dbg timeout 60 python tools/probe_tc.py --family $f --M $m --R 4 --tag "f$f M$m dbg$dbg $TAG" 2>&1 | tail -1
done; done
