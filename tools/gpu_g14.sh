OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_fullsize.py tests/test_gpu_allreduce.py tests/test_gpu_ipc.py -q -x --timeout 300 > $OUT/g14_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/g14_tests.log
BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline > $OUT/g14_bench.json 2> $OUT/g14_bench.err; echo "bench rc=$?"; tail -6 $OUT/g14_bench.err
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/g14_chainprobe.log 2>&1; head -3 $OUT/g14_chainprobe.log; tail -6 $OUT/g14_chainprobe.log
