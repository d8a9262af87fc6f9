OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_allreduce.py tests/test_gpu_ipc.py tests/test_gpu_multirank.py -q -x --timeout 700 -rs > $OUT/r2h_tests.log 2>&1; echo "tests rc=$?"; tail -8 $OUT/r2h_tests.log | cut -c1-300
BENCH_WATCHDOG=500 timeout 600 python bench.py --sweep "" --sym-sweep "" --no-kernels --no-cpu-baseline > $OUT/r2h_bench.json 2> $OUT/r2h_bench.err; echo "bench rc=$?"; grep -i 'allreduce\|error\|Trace' $OUT/r2h_bench.err | head
