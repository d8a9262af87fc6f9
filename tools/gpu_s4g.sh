for lib in "" old "" old; do
  W4A16_LIB="$lib" timeout 300 python tools/probe_fam.py --shapes qkv,down,c1 --M 8,64 --families 0,1 --bytes 1.5e9 --reps 3 2>&1 | grep -v "^\[" | sed "s/^/${lib:-new} /" | cut -c1-150
  W4A16_LIB="$lib" timeout 200 python tools/fwd_time.py --layers 16 --reps 15 --Ms 32,64 2>&1 | grep median
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_w4a8.py tests/test_gpu_lmhead.py -q -x --timeout 300 2>&1 | tail -2
