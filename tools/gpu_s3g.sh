OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_tree_attn.py -q -x --timeout 200 2>&1 | tail -2
for M in 8 61; do timeout 60 python tools/probe_attn.py --M $M --L 2048; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 3 -c 1 -f -o $OUT/prof_attn_s3g python tools/probe_attn.py --M 8 --L 2048 > /dev/null 2>&1; echo ncu rc=$?
ncu -i $OUT/prof_attn_s3g.ncu-rep --page raw --csv > $OUT/raw_attn_s3g.csv 2>/dev/null
ncu -i $OUT/prof_attn_s3g.ncu-rep --page details --csv > $OUT/details_attn_s3g.csv 2>/dev/null
