#!/bin/bash
# Cost experiments on the mma.sync consumer (libw4a16_exp<N>.so builds, -DW4_MA_EXP=N): compute-only (dbg 2).
for e in ${EXPS:-0 1 2 4 8 15}; do for fm in ${FMS:-"0:8"}; do f=${fm%%:*}; m=${fm##*:}
  W4A16_LIB=exp$e W4A16_MMA_DEBUG=2 timeout 60 python tools/probe_tc.py --family $f --M $m --R 4 --tag "exp$e f$f M$m dbg2" 2>&1 | tail -1 | cut -c1-120
done; done
