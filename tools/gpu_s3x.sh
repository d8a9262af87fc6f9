W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 300 python tools/probe_chain.py --M 8 --layers 8 2>&1 | tail -6
