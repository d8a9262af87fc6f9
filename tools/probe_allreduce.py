#!/usr/bin/env python
"""Cost of the in-chain ALLREDUCE op (include/w4a16.h) on one GPU: the Llama-3-70B-shaped stack of
--layers layers as one chain, with and without an ALLREDUCE after every O and down GEMM, over a world-1
group (flag store + system fences + flag waits + the reduce pass over the partial: everything but the
NVLink reads of peers' partials). Also --world T simulated ranks side by side (each on SMs/T; the stack
shards are tp = 1 shapes, so this measures protocol overhead at T, not a tp = T forward)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22179_b200 as w4
from paper_2505_22179_b200 import tp
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=16)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--Ms", default="1,8,16")
a = ap.parse_args()
mat_id = {n: i for i, n in enumerate(tp.MATRICES)}
st = tp.VerifyStack(tp.LLAMA3_70B, a.layers, 16, lambda l, n, K, N, out: synth.gpu(0, synth.tensor_id(l, mat_id[n], 0), synth.WEIGHT, K, N, out=out))
g = w4.PeerGroup.simulated(1, 1 << 22, 2 * a.layers, device="cuda")[0]
H = tp.LLAMA3_70B.hidden
P_o, P_d = g.alloc(16, H), g.alloc(16, H)
red_o, red_d = torch.empty(16, H, dtype=torch.float16, device="cuda"), torch.empty(16, H, dtype=torch.float16, device="cuda")


def timed(ch):
    for _ in range(3):
        ch()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ch(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


for M in [int(x) for x in a.Ms.split(",")]:
    plain, fused = [], []
    for L in st.layers:
        qa, qb = st._layer_ops(L, M)
        plain += qa + qb
        fused += [qa[0], ("gemm", st.q_part(M), L["o"], P_o[:M]), ("allreduce", P_o[:M], red_o[:M], g),
                  qb[0], qb[1], ("gemm", st.act[:M], L["down"], P_d[:M]), ("allreduce", P_d[:M], red_d[:M], g)]
    t0 = timed(w4.Chain(plain, M))
    t1 = timed(w4.Chain(fused, M))
    print(f"M={M} layers={a.layers}: chain {t0:.1f} us, with {2 * a.layers} ALLREDUCE ops (world 1) {t1:.1f} us "
          f"-> {(t1 - t0) / (2 * a.layers):.2f} us per op")
