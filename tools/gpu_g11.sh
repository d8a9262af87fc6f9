OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 -k "verify_stack or tp2" > $OUT/g11_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/g11_tests.log
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/g11_chain.log 2>&1; tail -8 $OUT/g11_chain.log
