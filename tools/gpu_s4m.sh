timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -3
for r in 1 2; do timeout 200 python tools/fwd_time.py --layers 16 --reps 15 --Ms 24,32,64 2>&1 | grep median; done
