timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "3" 2>&1 | tail -4
for lib in ""; do W4A16_LIB="$lib" timeout 300 python tools/probe_fam.py --shapes gate_up,down,qkv --M 1,8,16 --families 3 --bytes 1.5e9 --reps 3 2>&1 | grep -v "^\[" | cut -c1-200; done
