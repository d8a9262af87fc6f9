OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 700 > $OUT/r2w_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/r2w_tests.log
BENCH_WATCHDOG=300 timeout 400 python bench.py --sweep 1,8,16 --sym-sweep "" --no-kernels --no-lm-head --no-cpu-baseline 2>&1 >/dev/null | grep -E 'sweep'
timeout 200 python tools/probe_w4a8.py --Ms 1,8,16
