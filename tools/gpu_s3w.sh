for rep in 1 2; do for lib in "" df; do
  W4A16_LIB="$lib" timeout 200 python tools/fwd_time.py --layers 16 --reps 15 --Ms 24,32,64 2>&1 | grep median
done; done
W4A16_LIB=df timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "tc or fam or M64 or 64" 2>&1 | tail -2
