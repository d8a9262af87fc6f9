for r in 1 2; do for g in "" 1; do echo "glue=$g"; W4A16_AB_GLUE=$g timeout 200 python tools/fwd_time.py --layers 16 --reps 15 --Ms 24,32,64 2>&1 | grep median; done; done
