OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | tail -1
BENCH_WATCHDOG=800 timeout 1000 python bench.py > $OUT/bench_r02b.json 2> $OUT/bench_r02b.err; echo "bench rc=$?"; tail -2 $OUT/bench_r02b.err | cut -c1-200
