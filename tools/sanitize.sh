#!/bin/bash
# compute-sanitizer over small GPU parity cases (SURVEY §4 tier T4): memcheck (out-of-bounds / misaligned
# accesses), racecheck (shared-memory hazards) and synccheck (barrier misuse) on the W4A16 kernels.
OUT=gpurun_out; mkdir -p $OUT
SEL='test_gemm_config1_tolerance and (M-1- or M-16- or M-17-) or test_pack_bit_exact and 128 or test_accept_golden or one_hot'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -x -q -k "$SEL" > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_$tool.log | tail -2
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_chain.py -x -q \
    -k "independent or rejects" > $OUT/sanitize_chain.log 2>&1; echo "chain memcheck rc=$?"; grep -E "ERROR SUMMARY|passed" $OUT/sanitize_chain.log | tail -2
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_tree_attn.py -x -q \
    -k "not full_size and not 61 and not 49" > $OUT/sanitize_f23.log 2>&1; echo "f2/f3 memcheck rc=$?"; grep -E "ERROR SUMMARY|passed" $OUT/sanitize_f23.log | tail -2
# the publisher-warp handshake and the ALLREDUCE op (world 1 only: the sanitizer serialises kernels, so
# simulated ranks side by side would wait for each other until the 10 s trap)
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_chain.py tests/test_gpu_allreduce.py -x -q \
      -k "independent or (simulated_ranks and 1-8-0)" > $OUT/sanitize_chain_$tool.log 2>&1; echo "chain $tool rc=$?"; grep -E "ERROR SUMMARY|passed" $OUT/sanitize_chain_$tool.log | tail -2
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_w4a8.py -x -q -k "1024 or quant" \
    > $OUT/sanitize_w4a8.log 2>&1; echo "w4a8 memcheck rc=$?"; grep -E "ERROR SUMMARY|passed" $OUT/sanitize_w4a8.log | tail -2
