OUT=gpurun_out; mkdir -p $OUT
for d in 16 20 0; do W4A16_TP_DEBUG=$d timeout 100 python tools/probe_fam.py --shapes gate_up --M 8,16 --families 3 --bytes 1e9 | sed "s/^/dbg=$d /"; done > $OUT/g8_probe.log 2>&1
W4A16_MMA_DEBUG=2 timeout 100 python tools/probe_fam.py --shapes gate_up --M 8 --families 0 --bytes 1e9 | sed "s/^/famA-noload /" >> $OUT/g8_probe.log 2>&1
cat $OUT/g8_probe.log
