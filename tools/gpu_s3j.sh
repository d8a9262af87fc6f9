for c in 1 2 3 4 6; do for M in 8 61; do echo -n "cps>=$c "; W4A16_TA_CPS=$c timeout 60 python tools/probe_attn.py --M $M --L 2048; done; done
