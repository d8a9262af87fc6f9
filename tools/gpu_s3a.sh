OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_s3a.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_s3a.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 700 > $OUT/pytest_gpu_s3a.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_s3a.log
BENCH_WATCHDOG=800 timeout 1000 python bench.py > $OUT/bench_s3a.json 2> $OUT/bench_s3a.err; echo "bench rc=$?"; tail -3 $OUT/bench_s3a.err | cut -c1-300
