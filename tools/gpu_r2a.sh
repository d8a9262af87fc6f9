OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > $OUT/r2a_tests.log 2>&1; echo "tests rc=$?"; tail -4 $OUT/r2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2a_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/r2a_smoke.log
BENCH_WATCHDOG=700 timeout 900 python bench.py > $OUT/r2a_bench.json 2> $OUT/r2a_bench.err; echo "bench rc=$?"; tail -30 $OUT/r2a_bench.err | cut -c1-250
timeout 200 python tools/probe_fam.py --shapes gate_up,qkv,o,down,c1 --M 1,8,16,32,64 --families 0,1,2,3,4 --bytes 1e9 > $OUT/r2a_probe.log 2>&1; cat $OUT/r2a_probe.log | cut -c1-200
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/r2a_chainprobe.log 2>&1; tail -8 $OUT/r2a_chainprobe.log
