OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -q -x --timeout 200 > $OUT/r2b_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/r2b_tests.log
for lib in "" oc; do
W4A16_LIB=$lib timeout 200 python tools/probe_fam.py --shapes gate_up,qkv,o,down --M 1,8,16 --families 0,2 --bytes 1e9 2>&1 | sed "s/^/[${lib:-main}] /" | cut -c1-160
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline > $OUT/r2b_bench_${lib:-main}.json 2> $OUT/r2b_bench_${lib:-main}.err; echo "bench ${lib:-main} rc=$?"; grep sweep $OUT/r2b_bench_${lib:-main}.err
done
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/r2b_chainprobe.log 2>&1; tail -6 $OUT/r2b_chainprobe.log
