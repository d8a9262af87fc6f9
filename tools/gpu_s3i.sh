timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | grep -E "Error|assert|FAILED|err" | head -20
