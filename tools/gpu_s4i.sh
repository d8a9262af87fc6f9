timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | tail -1
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 300 python tools/probe_chain.py --M 8 --layers 8 2>&1 | grep -v "^$" | head -40
