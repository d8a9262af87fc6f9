OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "3 and not stress" > $OUT/g5_parity.log 2>&1; echo "parity rc=$?"; grep -E "passed|failed|FAILED" $OUT/g5_parity.log | head -20
for d in 0 15; do W4A16_TP_DEBUG=$d timeout 300 python tools/probe_fam.py --shapes gate_up --M 1,8,16,32,64 --families 3 --bytes 1e9 | sed "s/^/dbg=$d /"; done > $OUT/g5_probe.log 2>&1
W4A16_TP_DEBUG=256 timeout 300 python tools/probe_fam.py --shapes gate_up --M 8 --families 3 --bytes 1e9 > $OUT/g5_trace.log 2>&1
timeout 300 python tools/probe_fam.py --shapes gate_up,down --M 8 --families 0 --bytes 1e9 >> $OUT/g5_probe.log 2>&1
cat $OUT/g5_probe.log; head -40 $OUT/g5_trace.log
