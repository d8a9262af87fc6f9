#!/bin/bash
for m in 8 16; do timeout 60 python tools/probe_tc.py --family 0 --M $m --R 4 --tag famA_m$m 2>&1 | grep -v Warn; done
