OUT=gpurun_out; mkdir -p $OUT
for lib in base ch2 e1 e2 e4 e8 e3; do
for dbg in 0 2; do
W4A16_LIB=$lib W4A16_MMA_DEBUG=$dbg timeout 100 python tools/probe_fam.py --shapes gate_up --M 1,8,16 --families 0 --bytes 1e9 2>&1 | sed "s/^/[$lib dbg$dbg] /" | cut -c1-150
done; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 100 -k "stress or one_hot or tolerance" 2>&1 | tail -2
W4A16_LIB=ch2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 100 -k "stress or one_hot or tolerance" 2>&1 | tail -2
