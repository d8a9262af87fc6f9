#!/bin/bash
# A/B of the tcgen05 family: the default library vs variant libraries libw4a16_<name>.so
# (LIBS="diag v1 ..." selects them; build the B sides first). MS selects the token widths.
for lib in "" ${LIBS:-diag}; do for m in ${MS:-16 32 64}; do
  W4A16_LIB="$lib" timeout 60 python tools/probe_tc.py --family 1 --M $m --R 4 --tag "${lib:-main} tc M$m" 2>&1 | tail -1 | cut -c1-110
done; done
