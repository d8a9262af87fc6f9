OUT=gpurun_out; mkdir -p $OUT
W4A16_LIB=diag W4A16_MMA_DEBUG=64 timeout 200 python tools/probe_chain.py --layers 8 --M 8 > $OUT/g9_chain.log 2>&1; echo rc=$?
cat $OUT/g9_chain.log
