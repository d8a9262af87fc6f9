for rep in 1 2; do for lib in acq ""; do
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep' | sed "s/^/[${lib:-new}] /"
done; done
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 2>&1 | tail -12
timeout 300 python -m pytest tests/test_gpu_chain.py tests/test_gpu_allreduce.py -q -x --timeout 100 2>&1 | tail -2
