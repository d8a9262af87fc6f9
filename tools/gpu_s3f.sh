OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | tail -3
for M in 8 61; do timeout 60 python tools/probe_attn.py --M $M --L 2048; done
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_fullsize.py -q -x --timeout 300 2>&1 | tail -2
