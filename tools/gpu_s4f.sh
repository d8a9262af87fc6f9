for rep in 1 2; do W4A16_LIB="" timeout 120 python tools/chain_time.py --layers 16 --reps 15 --Ms 1,8,16 2>&1 | grep median; done
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 700 2>&1 | tail -2
