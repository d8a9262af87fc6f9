OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do for lib in old ""; do
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep' | sed "s/^/[${lib:-new}] /"
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py tests/test_gpu_allreduce.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -q -x --timeout 700 > $OUT/r2l_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/r2l_tests.log
grep -B2 -A25 'Error\|FAILED' $OUT/r2l_tests.log | head -60
BENCH_WATCHDOG=500 timeout 600 python bench.py --sweep "" --sym-sweep "" --no-kernels --no-cpu-baseline > $OUT/r2l_bench.json 2> $OUT/r2l_bench.err; echo "bench rc=$?"; grep -i 'allreduce' $OUT/r2l_bench.err | head
