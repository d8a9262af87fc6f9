#!/bin/bash
# A/B of the mma.sync family: the default library vs libw4a16_diag.so (build the B side into it first).
for rep in 1 2; do
for lib in "" diag; do
  for fm in "0 8" "2 16" "0 1"; do set -- $fm
    W4A16_LIB="$lib" timeout 60 python tools/probe_tc.py --family $1 --M $2 --R 4 --tag "${lib:-main} f$1 M$2" 2>&1 | tail -1 | cut -c1-110
  done
done; done
