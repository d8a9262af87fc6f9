OUT=gpurun_out; mkdir -p $OUT
for cfg in "base 2" "base 0" "e3 2"; do set -- $cfg
W4A16_LIB=$1 W4A16_MMA_DEBUG=$2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a16_mma -s 3 -c 1 -f -o $OUT/prof_famA_$1_d$2 \
  python tools/probe_fam.py --shapes gate_up --M 8 --families 0 --bytes 6e8 --reps 1 > $OUT/ncu_famA_$1_d$2.log 2>&1; echo "ncu $1 $2 rc=$?"
ncu -i $OUT/prof_famA_$1_d$2.ncu-rep --page source --csv --print-source sass > $OUT/src_famA_$1_d$2.csv 2>/dev/null
ncu -i $OUT/prof_famA_$1_d$2.ncu-rep --page raw --csv > $OUT/raw_famA_$1_d$2.csv 2>/dev/null
done
