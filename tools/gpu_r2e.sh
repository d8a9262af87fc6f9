OUT=gpurun_out; mkdir -p $OUT
W4A16_LIB=g3 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -q -x --timeout 100 2>&1 | tail -2
for lib in "" g3; do
W4A16_LIB=$lib timeout 100 python tools/probe_fam.py --shapes gate_up,down,qkv --M 1,8,16 --families 0 --bytes 1e9 2>&1 | sed "s/^/[${lib:-main}] /" | cut -c1-150
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep sweep | sed "s/^/[${lib:-main}] /"
done
