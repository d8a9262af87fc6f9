OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/g1_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 1400 > $OUT/g1_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/g1_pytest.log
BENCH_WATCHDOG=700 timeout 900 python bench.py > $OUT/g1_bench.json 2> $OUT/g1_bench.err; echo "bench rc=$?"; tail -40 $OUT/g1_bench.err
