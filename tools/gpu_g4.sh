OUT=gpurun_out; mkdir -p $OUT
for d in 0 1 2 4 8 3 15; do W4A16_TP_DEBUG=$d timeout 300 python tools/probe_fam.py --shapes gate_up --M 8 --families 3 --bytes 1e9 | sed "s/^/dbg=$d /"; done > $OUT/g4_probe.log 2>&1
W4A16_TP_DEBUG=256 timeout 300 python tools/probe_fam.py --shapes gate_up --M 8 --families 3 --bytes 1e9 > $OUT/g4_trace.log 2>&1
W4A16_TP_DEBUG=257 timeout 300 python tools/probe_fam.py --shapes gate_up --M 8 --families 3 --bytes 1e9 > $OUT/g4_trace_nomma.log 2>&1
W4A16_TP_DEBUG=271 timeout 300 python tools/probe_fam.py --shapes gate_up --M 8 --families 3 --bytes 1e9 > $OUT/g4_trace_skel.log 2>&1
cat $OUT/g4_probe.log; head -40 $OUT/g4_trace.log
