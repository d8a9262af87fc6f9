for r in 1 2; do timeout 120 python tools/probe_w4a8.py 2>&1 | tail -3; done
timeout 300 python tools/probe_fam.py --shapes gate_up --M 8 --families 0 --bytes 1.5e9 --reps 3 2>&1 | grep -v "^\["
