#!/usr/bin/env python
"""Diagnostics: time one GEMM shape for both families, back-to-back over R distinct weight copies (CUDA graph).
Run under different W4A16_TC_DEBUG values to localise the tcgen05 pipeline bottleneck."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22179_b200 as w4
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=8192); ap.add_argument("--N", type=int, default=57344)
ap.add_argument("--M", type=int, default=16); ap.add_argument("--R", type=int, default=8)
ap.add_argument("--family", type=int, default=1); ap.add_argument("--tag", default="")
a = ap.parse_args()
lins = []
for r in range(a.R):
    W = synth.gpu(0, 100 + r, synth.WEIGHT, a.K, a.N)
    lins.append(w4.pack_linear(W)); del W
X = synth.gpu(0, 2, synth.ACT, a.M, a.K)
Y = torch.empty(a.M, a.N, dtype=torch.float16, device="cuda")
ws = w4.alloc_workspace(a.M, [(a.K, a.N)])
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for l in lins: l(X, Y, ws, s, family=a.family)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for l in lins: l(X, Y, ws, s, family=a.family)
for _ in range(3): g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record(); [g.replay() for _ in range(n)]; e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (n * a.R)
wb = lins[0].weight_bytes
print(json.dumps({"tag": a.tag, "dbg": os.environ.get("W4A16_TC_DEBUG", "0"), "K": a.K, "N": a.N, "M": a.M,
                  "family": a.family, "us": us, "GBps": wb / us / 1e3}))
if int(os.environ.get("W4A16_TC_DEBUG", "0")) & 256:
    import ctypes, numpy as np
    from paper_2505_22179_b200._lib import lib
    buf = np.zeros((16, 64), dtype=np.uint64)
    lib.w4a16_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)
    t0 = int(buf[0, 0])
    names = ["P_emptyok", "P_issued", "D_full", "D_aempty0", "D_afull0", "D_aempty1", "D_afull1", "M_full", "M_afull0",
             "M_issued0", "M_afull1", "M_issued1", "M_done0"]
    print("stage " + " ".join(f"{n:>9}" for n in names))
    for i in range(20):
        print(f"{i:5d} " + " ".join(f"{(int(buf[e, i]) - t0) if buf[e, i] else -1:9d}" for e in range(len(names))))
