OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "not fullsize" > $OUT/g2_parity.log 2>&1; echo "parity rc=$?"; tail -5 $OUT/g2_parity.log
timeout 600 python tools/probe_fam.py --shapes gate_up,qkv,o,down --M 1,8,16,32,64 --families 0,2,1,3 > $OUT/g2_probe.log 2>&1; echo "probe rc=$?"; cat $OUT/g2_probe.log | cut -c1-200
