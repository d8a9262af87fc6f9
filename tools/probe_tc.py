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
print(json.dumps({"tag": a.tag, "dbg": os.environ.get("W4A16_TC_DEBUG", "0") + "/" + os.environ.get("W4A16_MMA_DEBUG", "0"), "K": a.K, "N": a.N, "M": a.M,
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
if int(os.environ.get("W4A16_MMA_DEBUG", "0")) & 16:
    import ctypes, numpy as np
    from paper_2505_22179_b200._lib import lib
    buf = np.zeros((1024, 8), dtype=np.uint64)
    lib.w4a16_debug_trace_mma(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)
    G = int((buf[:, 0] > 0).sum())
    b = buf[:G].astype(np.int64)
    smid = b[:, 7].copy()
    t0 = b[:, 0].min()
    b[:, :7] -= t0
    q = lambda v: " ".join(f"{x:7.0f}" for x in np.percentile(v, [0, 10, 50, 90, 100]))
    print(f"CTAs {G}; ns percentiles 0/10/50/90/100")
    print("entry      ", q(b[:, 0])); print("first ready", q(b[:, 1])); print("loop done  ", q(b[:, 2])); print("exit       ", q(b[:, 3]))
    print("flush dur  ", q(b[:, 3] - b[:, 2])); print("loop dur   ", q(b[:, 2] - b[:, 1]))
    mid = b[:, 4] > 0
    if mid.any(): print("mid flush  ", q((b[:, 5] - b[:, 4])[mid]))
    ld = b[:, 2] - b[:, 1]
    for lo_, hi_ in ((0, 74), (74, 148)):
        sel = (smid >= lo_) & (smid < hi_)
        if sel.any(): print(f"smid {lo_}-{hi_}: loop dur", q(ld[sel]))
    order = np.argsort(ld)
    print("slowest CTAs (cta, smid, loop dur):", [(int(c), int(smid[c]), int(ld[c])) for c in order[-8:]])
    print("fastest CTAs:", [(int(c), int(smid[c]), int(ld[c])) for c in order[:8]])
    # CTA pairs sharing an SM
    from collections import defaultdict
    per = defaultdict(list)
    for c in range(G): per[int(smid[c])].append(c)
    cnt = np.bincount([len(v) for v in per.values()])
    print("CTAs per SM histogram:", cnt.tolist())
    if cnt.size < 3: sys.exit(0)
    fast = np.array([min(ld[c] for c in v) for v in per.values() if len(v) == 2])
    slow = np.array([max(ld[c] for c in v) for v in per.values() if len(v) == 2])
    done = np.array([max(b[c, 2] for c in v) for v in per.values()])
    ent = np.array([abs(b[v[0], 0] - b[v[1], 0]) for v in per.values() if len(v) == 2])
    print("per-SM faster CTA loop dur", q(fast)); print("per-SM slower CTA loop dur", q(slow))
    print("per-SM last loop done     ", q(done)); print("per-SM entry skew         ", q(ent))
