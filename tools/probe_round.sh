#!/bin/bash
for f in 0 2; do for m in 1 8 16; do timeout 60 python tools/probe_tc.py --family $f --M $m --R 4 --tag fam${f}_m$m 2>&1 | grep -v Warn; done; done
