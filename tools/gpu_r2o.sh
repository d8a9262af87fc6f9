timeout 900 python -m pytest tests/test_gpu_w4a8.py -q -x --timeout 120 2>&1 | tail -3
timeout 200 python tools/probe_w4a8.py --Ms 1,8,16,64
