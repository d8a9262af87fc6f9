OUT=gpurun_out; mkdir -p $OUT
for d in 0 15; do W4A16_TP_DEBUG=$d timeout 300 python tools/probe_fam.py --shapes gate_up --M 1,8,16 --families 3 --bytes 1e9 | sed "s/^/dbg=$d /"; done > $OUT/g6_probe.log 2>&1
W4A16_TP_DEBUG=256 timeout 300 python tools/probe_fam.py --shapes gate_up --M 8 --families 3 --bytes 1e9 > $OUT/g6_trace.log 2>&1
cat $OUT/g6_probe.log; head -30 $OUT/g6_trace.log
