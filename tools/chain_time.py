#!/usr/bin/env python
"""A/B timing of the persistent chain (whole Llama-3-70B-shaped stack of --layers layers, tp = 1): median of
--reps back-to-back runs per M. W4A16_LIB=<name> selects libw4a16_<name>.so (tools only)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_22179_b200 import tp
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=16)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--Ms", default="1,8,16")
ap.add_argument("--tag", default=os.environ.get("W4A16_LIB", "main") or "main")
a = ap.parse_args()
mat_id = {n: i for i, n in enumerate(tp.MATRICES)}
st = tp.VerifyStack(tp.LLAMA3_70B, a.layers, 64, lambda l, n, K, N, out: synth.gpu(0, synth.tensor_id(l, mat_id[n], 0), synth.WEIGHT, K, N, out=out))
for M in [int(x) for x in a.Ms.split(",")]:
    ch = st.chains(M)[0]
    for _ in range(3):
        ch()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ch(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    gb = st.weight_bytes / 1e9
    med = ts[len(ts) // 2]
    print(f"{a.tag} M={M} layers={a.layers}: median {med:.1f} us  ({gb / med * 1e6 / 1e3:.3f} TB/s)  min {ts[0]:.1f}")
