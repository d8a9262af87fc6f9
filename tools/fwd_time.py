#!/usr/bin/env python
"""A/B timing of the verify forward (Llama-3-70B-shaped stack of --layers layers, tp = 1) as a captured CUDA
graph (VerifyStack.capture: chain at M <= 16, op-by-op tcgen05 launches above): median of --reps replays per M.
W4A16_LIB=<name> selects libw4a16_<name>.so (tools only)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_22179_b200 import tp
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=16)
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--Ms", default="24,32,64")
ap.add_argument("--tag", default=os.environ.get("W4A16_LIB", "main") or "main")
a = ap.parse_args()
mat_id = {n: i for i, n in enumerate(tp.MATRICES)}
st = tp.VerifyStack(tp.LLAMA3_70B, a.layers, 64, lambda l, n, K, N, out: synth.gpu(0, synth.tensor_id(l, mat_id[n], 0), synth.WEIGHT, K, N, out=out))
for M in [int(x) for x in a.Ms.split(",")]:
    g = st.capture(M)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{a.tag} M={M} layers={a.layers}: median {med:.1f} us  ({st.weight_bytes / 1e9 / med * 1e6 / 1e3:.3f} TB/s)  min {ts[0]:.1f}")
