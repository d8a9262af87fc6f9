OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_allreduce.py tests/test_gpu_ipc.py tests/test_gpu_chain.py -q -x --timeout 300 > $OUT/r2f_tests.log 2>&1; echo "tests rc=$?"; tail -15 $OUT/r2f_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 -k "tp2 or fused or stack" > $OUT/r2f_full.log 2>&1; echo "full rc=$?"; tail -3 $OUT/r2f_full.log
BENCH_WATCHDOG=500 timeout 600 python bench.py --sweep "" --sym-sweep "" --no-kernels --no-cpu-baseline > $OUT/r2f_bench.json 2> $OUT/r2f_bench.err; echo "bench rc=$?"; grep -i 'allreduce\|error\|Trace' $OUT/r2f_bench.err | head
