timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -q -x --timeout 200 2>&1 | tail -1
for rep in 1 2; do for lib in nopair ""; do
W4A16_LIB=$lib BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep' | sed "s/^/[${lib:-pair}] /"
done; done
for lib in nopair ""; do W4A16_LIB=$lib timeout 100 python tools/probe_fam.py --shapes gate_up,qkv,down --M 8 --families 0 --bytes 1e9 2>&1 | sed "s/^/[${lib:-pair}] /" | cut -c1-140; done
