OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "3 or stress" > $OUT/g3_parity.log 2>&1; echo "parity rc=$?"; grep -E "passed|failed|FAILED" $OUT/g3_parity.log | head -20
timeout 600 python tools/probe_fam.py --shapes gate_up,down,qkv --M 1,8,16,32,64 --families 0,3 > $OUT/g3_probe.log 2>&1; echo "probe rc=$?"; cat $OUT/g3_probe.log | cut -c1-150
