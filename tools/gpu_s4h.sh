timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | tail -1
for r in 1 2; do for M in 8 61; do timeout 60 python tools/probe_attn.py --M $M --L 2048; done; done
