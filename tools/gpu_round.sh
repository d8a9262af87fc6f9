#!/bin/bash
# One gpurun call: parity tests, smoke, bench (N=1), ncu launch list + full capture of the top kernel.
# Usage (from repo root, on the GPU box): bash tools/gpu_round.sh <tag>
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 $OUT/bench_$TAG.json; tail -5 $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --layers 4 --steps 2 --warmup 1 --sweep "" --no-cpu-baseline > $OUT/bench_ncu_$TAG.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a16 -s 2 -c 1 -f -o $OUT/prof_gateup_$TAG \
    python tools/profile_gemm.py --K 8192 --N 57344 --M 16 > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
