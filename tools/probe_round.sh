#!/bin/bash
for fm in "0 1" "0 8" "0 16" "2 16"; do set -- $fm
timeout 60 python tools/probe_tc.py --family $1 --M $2 --R 4 --tag GU_fam${1}_m${2} 2>&1 | grep -v Warn
done
for d in 2 34; do W4A16_MMA_DEBUG=$d timeout 60 python tools/probe_tc.py --family 0 --M 16 --R 4 --tag GU_fam0_m16_d$d 2>&1 | grep -v Warn; done
for fm in "0 8" "0 16"; do set -- $fm
timeout 60 python tools/probe_tc.py --K 8192 --N 8192 --family $1 --M $2 --R 16 --tag O_fam${1}_m${2} 2>&1 | grep -v Warn
done
