#!/bin/bash
# Cost experiments on the mma.sync consumer: build libw4a16_exp<N>.so with -DW4A16_MMA_DIAG=1 -DW4_MA_EXP=N
# (see gemm_mma.cu), then time compute only (W4A16_MMA_DEBUG=2: loads skipped).
for e in ${EXPS:-0 1 2 4 8 15}; do for fm in ${FMS:-"0:8"}; do f=${fm%%:*}; m=${fm##*:}
  W4A16_LIB=exp$e W4A16_MMA_DEBUG=2 timeout 60 python tools/probe_tc.py --family $f --M $m --R 4 --tag "exp$e f$f M$m dbg2" 2>&1 | tail -1 | cut -c1-120
done; done
