OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a16_mma -s 70 -c 1 -f -o $OUT/prof_chain_r02 \
    python bench.py --layers 8 --steps 1 --warmup 3 --sweep "" --sym-sweep "" --no-cpu-baseline --no-kernels --no-lm-head > $OUT/ncu_chain_r02.log 2>&1; echo "ncu chain rc=$?"
ncu -i $OUT/prof_chain_r02.ncu-rep --page raw --csv > $OUT/raw_chain_r02.csv 2>/dev/null
ncu -i $OUT/prof_chain_r02.ncu-rep --page source --csv --print-source sass > $OUT/src_chain_r02.csv 2>/dev/null
timeout 600 python tools/probe_attn.py > $OUT/attn_base.log 2>&1; tail -8 $OUT/attn_base.log
