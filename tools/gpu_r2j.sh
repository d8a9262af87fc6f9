for rep in 1 2; do for lib in old noar noarpub pubold ""; do
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 8 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep' | sed "s/^/[${lib:-new}] /"
done; done
