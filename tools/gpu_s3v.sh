for rep in 1 2; do for lib in "" old; do
  W4A16_LIB="$lib" timeout 200 python tools/fwd_time.py --layers 16 --reps 15 --Ms 24,32,64 2>&1 | grep median
done; done
