#!/bin/bash
# tcgen05 family cost decomposition on the gate-up shape: W4A16_TC_DEBUG bit0 skip MMA, bit1 skip dequant,
# bit2 skip the activation TMA.
for m in ${MS:-16 64}; do for dbg in ${DBGS:-0 1 2 3}; do
  W4A16_TC_DEBUG=$dbg timeout 60 python tools/probe_tc.py --family 1 --M $m --R 4 --tag "tc M$m dbg$dbg" 2>&1 | tail -1
done; done
