OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2; do for lib in old ""; do
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep|e2e' | sed "s/^/[${lib:-new}] /"
done; done
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/r2i_chainprobe.log 2>&1; tail -6 $OUT/r2i_chainprobe.log
