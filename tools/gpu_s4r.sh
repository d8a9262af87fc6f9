for rep in 1 2; do for lib in "" os0; do
  W4A16_LIB="$lib" timeout 120 python tools/chain_time.py --layers 16 --reps 15 --Ms 1,8,16 2>&1 | grep median
done; done
W4A16_LIB=os0 timeout 900 python -m pytest tests/test_gpu_chain.py -q -x --timeout 300 2>&1 | tail -2
