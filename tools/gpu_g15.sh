OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $OUT/g15_tests.log 2>&1; echo "tests rc=$?"; tail -4 $OUT/g15_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/g15_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/g15_smoke.log
BENCH_WATCHDOG=700 timeout 900 python bench.py > $OUT/g15_bench.json 2> $OUT/g15_bench.err; echo "bench rc=$?"; tail -40 $OUT/g15_bench.err | cut -c1-250
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/g15_chainprobe.log 2>&1; tail -5 $OUT/g15_chainprobe.log
