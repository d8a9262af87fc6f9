for mu in 0 8 16 24 32; do
W4A16_MMA_MIN_UNITS=$mu timeout 100 python tools/probe_fam.py --shapes c1,qkv,o --M 8 --families 0 --bytes 1e9 2>&1 | sed "s/^/[mu$mu] /" | cut -c1-140
done
