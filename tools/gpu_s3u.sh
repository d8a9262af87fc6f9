OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_s3u.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_s3u.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 700 > $OUT/pytest_gpu_s3u.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_s3u.log
BENCH_WATCHDOG=800 timeout 1000 python bench.py > $OUT/bench_s3u.json 2> $OUT/bench_s3u.err; echo "bench rc=$?"; tail -2 $OUT/bench_s3u.err | cut -c1-200
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 300 python tools/probe_chain.py --M 8 --layers 8 > $OUT/probe_chain_s3u.log 2>&1; echo "probe rc=$?"
