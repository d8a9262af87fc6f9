OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | tail -2
for M in 8 61 1 16; do timeout 60 python tools/probe_attn.py --M $M --L 2048; done
