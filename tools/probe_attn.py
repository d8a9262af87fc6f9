#!/usr/bin/env python
"""Diagnostics: time w4a16_tree_attention (f2) at a given verify width / context (70B head layout)."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_22179_b200 as w4
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=61); ap.add_argument("--L", type=int, default=2048)
ap.add_argument("--Hq", type=int, default=64); ap.add_argument("--Hkv", type=int, default=8)
a = ap.parse_args()
D = 128
Q = synth.gpu(0, 1, synth.ACT, a.M, a.Hq * D).view(a.M, a.Hq, D)
K = synth.gpu(0, 2, synth.ACT, a.L + a.M, a.Hkv * D).view(a.L + a.M, a.Hkv, D)
V = synth.gpu(0, 3, synth.ACT, a.L + a.M, a.Hkv * D).view(a.L + a.M, a.Hkv, D)
_, par = synth.eagle_tree(np.random.default_rng(0), a.M - 1, 6)
par = torch.tensor(par, dtype=torch.int32, device="cuda")
O = torch.empty(a.M, a.Hq, D, dtype=torch.float16, device="cuda")
ws = torch.zeros(w4.w4a16_tree_attention_workspace_bytes(a.M, a.L, a.Hq, a.Hkv, D), dtype=torch.uint8, device="cuda")
for _ in range(3):
    w4.w4a16_tree_attention(Q, K, V, par, O, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    w4.w4a16_tree_attention(Q, K, V, par, O, ws)
e1.record(); torch.cuda.synchronize()
eager = e0.elapsed_time(e1) * 1e3 / 20
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(20):
        w4.w4a16_tree_attention(Q, K, V, par, O, ws, stream=s)
with torch.cuda.stream(s):
    g.replay()
    torch.cuda.synchronize()
    e0.record(s); g.replay(); e1.record(s)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 20
kv = 2 * (a.L + a.M) * a.Hkv * D * 2
print(json.dumps({"M": a.M, "L": a.L, "us_eager": eager, "us_graph": us, "kv_GBps": kv / us / 1e3}))
