#!/bin/bash
# A/B of the tcgen05 family: the default library vs libw4a16_diag.so (build the B side into it first).
for lib in "" diag; do for m in 16 32 64; do
  W4A16_LIB="$lib" timeout 60 python tools/probe_tc.py --family 1 --M $m --R 4 --tag "${lib:-main} tc M$m" 2>&1 | tail -1 | cut -c1-110
done; done
