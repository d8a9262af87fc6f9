timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | tail -2
for M in 8 61; do timeout 120 python tools/probe_attn.py --M $M; W4A16_TA_PARTIALS=1 timeout 120 python tools/probe_attn.py --M $M | sed 's/^/[partials] /'; done
