OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 100 -k "not stress" > $OUT/g13_parity.log 2>&1; echo "parity rc=$?"; tail -2 $OUT/g13_parity.log
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_allreduce.py -q -x --timeout 200 > $OUT/g13_chain.log 2>&1; echo "chain rc=$?"; tail -2 $OUT/g13_chain.log
timeout 100 python tools/probe_fam.py --shapes gate_up,qkv,down --M 1,8,16 --families 0,2 --bytes 1e9 > $OUT/g13_probe.log 2>&1; cat $OUT/g13_probe.log
BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline > $OUT/g13_bench.json 2> $OUT/g13_bench.err; echo "bench rc=$?"; tail -6 $OUT/g13_bench.err
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/g13_chainprobe.log 2>&1; tail -6 $OUT/g13_chainprobe.log
