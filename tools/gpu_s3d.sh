OUT=gpurun_out; mkdir -p $OUT
for dbg in 64 66 65; do
W4A16_LIB=diag W4A16_MMA_DEBUG=$dbg timeout 300 python tools/probe_chain.py --M 8 --layers 8 > $OUT/probe_chain_s3d_$dbg.log 2>&1; echo "probe $dbg rc=$?"
head -12 $OUT/probe_chain_s3d_$dbg.log; sed -n '/per op/,/^$/p' $OUT/probe_chain_s3d_$dbg.log
done
