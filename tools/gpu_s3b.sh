OUT=gpurun_out; mkdir -p $OUT
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 300 python tools/probe_chain.py --M 8 --layers 8 > $OUT/probe_chain_s3b.log 2>&1; echo "probe rc=$?"
cat $OUT/probe_chain_s3b.log | tail -40
