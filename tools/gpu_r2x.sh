timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py tests/test_gpu_w4a8.py -q -x --timeout 200 2>&1 | tail -2
for rep in 1 2; do
BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep'
done
timeout 100 python tools/probe_fam.py --shapes gate_up,qkv --M 8 --families 0 --bytes 1e9 2>&1 | cut -c1-140
