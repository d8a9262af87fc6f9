#!/usr/bin/env python
"""Launch a few w4a16_gemm calls of one shape for ncu (not a benchmark; numbers under ncu are never reported).

  ncu --set full --clock-control none --import-source on -k regex:gemm_w4a16 -s 2 -c 1 -o gpurun_out/prof \
      python tools/profile_gemm.py --K 8192 --N 57344 --M 16
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2505_22179_b200 as w4  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=8192)
ap.add_argument("--N", type=int, default=57344)
ap.add_argument("--M", type=int, default=16)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--mode", default="asym")
a = ap.parse_args()
mode = w4.W4A16_SYM if a.mode == "sym" else w4.W4A16_ASYM
W = synth.gpu(0, 1, synth.WEIGHT, a.K, a.N)
lin = w4.pack_linear(W, mode=mode)
del W
X = synth.gpu(0, 2, synth.ACT, a.M, a.K)
Y = torch.empty(a.M, a.N, dtype=torch.float16, device="cuda")
ws = w4.alloc_workspace(a.M, [(a.K, a.N)])
for _ in range(a.iters):
    lin(X, Y, ws)
torch.cuda.synchronize()
print("ok", lin.weight_bytes)
