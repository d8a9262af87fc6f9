OUT=gpurun_out; mkdir -p $OUT
W4A16_MC_DEBUG=1 timeout 60 python -c "
import torch, paper_2505_22179_b200 as w4
print('supported', w4.PeerGroup.mc_supported())
g = w4.PeerGroup.mc(1 << 22, 4)
print('mc ok', hex(g.desc.mc_base), g.kind)
g.close(); print('closed')
" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_allreduce.py tests/test_gpu_ipc.py -q -x --timeout 300 > $OUT/r2g_tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/r2g_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 > $OUT/r2g_full.log 2>&1; echo "full rc=$?"; tail -3 $OUT/r2g_full.log
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 700 > $OUT/r2g_mr.log 2>&1; echo "multirank rc=$?"; tail -30 $OUT/r2g_mr.log | cut -c1-300
