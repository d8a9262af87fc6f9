#!/usr/bin/env python
"""W4A8 (f4) timing vs W4A16 on one GEMM shape: quantise + GEMM back to back in a CUDA graph."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22179_b200 as w4
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=8192)
ap.add_argument("--N", type=int, default=57344)
ap.add_argument("--Ms", default="1,8,16,64")
a = ap.parse_args()
pl = w4.pack_linear(synth.gpu(0, 1, synth.WEIGHT, a.K, a.N), mode=w4.W4A16_SYM)
wb = pl.weight_bytes if hasattr(pl, "weight_bytes") else a.K * a.N // 2 + (a.K // 128) * a.N * 2
s = torch.cuda.Stream()
for M in [int(x) for x in a.Ms.split(",")]:
    X = synth.gpu(0, 2, synth.ACT, M, a.K)
    Xq = torch.empty(M, a.K, dtype=torch.int8, device="cuda")
    sx = torch.empty(M, dtype=torch.float32, device="cuda")
    xs = torch.empty(M, a.K // 128, dtype=torch.int32, device="cuda")
    ws = torch.zeros(w4.w4a8_workspace_bytes(M, a.K, a.N), dtype=torch.uint8, device="cuda")
    Y = torch.empty(M, a.N, dtype=torch.float16, device="cuda")
    ws16 = w4.alloc_workspace(M, [(a.K, a.N)])
    res = {}
    for name in ("w4a8", "w4a8_famA", "w4a8_r1", "w4a8_gemm_only", "w4a16"):
        if name == "w4a8_famA" and M > 16:
            continue
        def step():
            if name.startswith("w4a8"):
                impl = {"w4a8": 0, "w4a8_famA": 1, "w4a8_r1": 2, "w4a8_gemm_only": 0}[name]
                if name != "w4a8_gemm_only":
                    w4.w4a8_quantize_act(X, Xq, sx, xs, stream=s)
                w4.w4a8_gemm(Xq, sx, xs, pl.packed, Y, ws, stream=s, impl=impl)
            else:
                pl(X, Y, ws16, stream=s)
        with torch.cuda.stream(s):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            g.replay()
            e0.record(s)
            for _ in range(5):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 50
        res[name] = us
    print(f"M={M} K={a.K} N={a.N}: " + " | ".join(f"{k} {v:.1f} us ({wb / v / 1e6:.2f} TB/s)" for k, v in res.items()))
