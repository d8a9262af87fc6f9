#!/usr/bin/env python
"""A/B of the chain's mma.sync families (0 = offset codes, 2 = scales in A) at given widths, 16-layer 70B stack."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22179_b200 as w4
from paper_2505_22179_b200 import tp
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=16)
ap.add_argument("--Ms", default="8,9,12,16")
a = ap.parse_args()
mat_id = {n: i for i, n in enumerate(tp.MATRICES)}
st = tp.VerifyStack(tp.LLAMA3_70B, a.layers, 64, lambda l, n, K, N, out: synth.gpu(0, synth.tensor_id(l, mat_id[n], 0), synth.WEIGHT, K, N, out=out))
for M in [int(x) for x in a.Ms.split(",")]:
    for fam in (0, 2):
        ops = [op for L in st.layers for seg in st._layer_ops(L, M) for op in seg]
        try:
            ch = w4.Chain(ops, M, family=fam)
        except w4.W4A16Error as e:
            print(M, fam, "n/a", e); continue
        for _ in range(3):
            ch()
        ts = []
        for _ in range(15):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ch(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"M={M} family={fam}: median {ts[len(ts)//2]:.1f} us ({st.weight_bytes / ts[len(ts)//2] / 1e6:.3f} TB/s)")
