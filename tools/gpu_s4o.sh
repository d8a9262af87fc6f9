timeout 600 python -m pytest tests/test_gpu_chain.py -q -x --timeout 300 2>&1 | tail -3
