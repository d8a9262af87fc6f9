for rep in 1 2; do for lib in old ""; do
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,24,64 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep' | sed "s/^/[${lib:-new}] /"
done; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 100 -k silu 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 300 -k "stack" 2>&1 | tail -1
