#!/bin/bash
# One gpurun call: smoke, parity tests, bench (N=1), ncu launch list + full captures of the top kernels.
# Usage (from repo root, on the GPU box): bash tools/gpu_round.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 700 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
BENCH_WATCHDOG=800 timeout 1000 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -3 $OUT/bench_$TAG.err
# launch list of the bench command (4 layers): every launch with its device time (cold, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --layers 4 --steps 3 --warmup 3 --sweep "" --sym-sweep "" --no-cpu-baseline --no-kernels --no-lm-head > $OUT/bench_ncu_$TAG.log 2>&1; echo "ncu list rc=$?"
# full capture of the dominant kernel: the persistent chain (8-layer stack, headline M=8)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a16_mma -s 70 -c 1 -f -o $OUT/prof_chain_$TAG \
    python bench.py --layers 8 --steps 1 --warmup 3 --sweep "" --sym-sweep "" --no-cpu-baseline --no-kernels --no-lm-head > $OUT/ncu_chain_$TAG.log 2>&1; echo "ncu chain rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a16_mma -s 3 -c 1 -f -o $OUT/prof_famA_$TAG \
    python tools/probe_fam.py --shapes gate_up --M 8 --families 0 --bytes 6e8 --reps 1 > $OUT/ncu_famA_$TAG.log 2>&1; echo "ncu famA rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a16_tc -s 3 -c 1 -f -o $OUT/prof_famB_$TAG \
    python tools/probe_fam.py --shapes gate_up --M 64 --families 1 --bytes 6e8 --reps 1 > $OUT/ncu_famB_$TAG.log 2>&1; echo "ncu famB rc=$?"
for k in chain famA famB; do
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page raw --csv > $OUT/raw_${k}_$TAG.csv 2>/dev/null
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/src_${k}_$TAG.csv 2>/dev/null
done
# f2: the tree-attention kernel at the bench's configuration (M = 8, L = 2048, 70B heads)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 3 -c 1 -f -o $OUT/prof_attn_$TAG \
    python tools/probe_attn.py --M 8 --L 2048 > $OUT/ncu_attn_$TAG.log 2>&1; echo "ncu attn rc=$?"
ncu -i $OUT/prof_attn_$TAG.ncu-rep --page raw --csv > $OUT/raw_attn_$TAG.csv 2>/dev/null
