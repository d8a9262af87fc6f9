#!/usr/bin/env python
"""Diagnostics: per-op timeline of the persistent chain kernel (needs the diag build: make diag;
W4A16_LIB=diag W4A16_MMA_DEBUG=64). Prints, per op kind, medians over layers of: the op's span (first CTA
start -> last CTA done), the CTAs' wait before their first stage, compute time, flush time, and skew."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_22179_b200 as w4
from paper_2505_22179_b200 import tp
from paper_2505_22179_b200._lib import lib
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=8)
ap.add_argument("--layers", type=int, default=8)
a = ap.parse_args()
mat_id = {n: i for i, n in enumerate(tp.MATRICES)}
st = tp.VerifyStack(tp.LLAMA3_70B, a.layers, 64, lambda l, n, K, N, out: synth.gpu(0, synth.tensor_id(l, mat_id[n], 0), synth.WEIGHT, K, N, out=out),
                    calibrate=synth.gpu(0, 9, synth.ACT, 8, 8192))
synth.gpu(0, synth.tensor_id(0xFFF, 1, 0), synth.ACT, st.x_in.shape[0], st.x_in.shape[1], out=st.x_in)
ch = st.chains(a.M)[0]
for _ in range(3):
    ch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
lib.w4a16_debug_prod_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
lib.w4a16_debug_prod_trace(None, 0, 1)
torch.cuda.synchronize()
e0.record(); ch(); e1.record(); torch.cuda.synchronize()
print(f"chain {a.layers} layers M={a.M}: {e0.elapsed_time(e1) * 1e3:.1f} us")
G, NOPS = 296, 512
buf = np.zeros((G, NOPS, 8), dtype=np.uint64)
lib.w4a16_debug_op_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.w4a16_debug_op_trace(buf.ctypes.data, buf.nbytes) == 0
n = ch.n
G = int((buf[:, 0, 0] > 0).sum())   # CTAs of this chain
b = buf[:G, :n, :].astype(np.int64)
t0 = b[:, 0, 0].min()
b -= t0
pt = np.zeros((296, 512), dtype=np.uint64)
lib.w4a16_debug_prod_trace(pt.ctypes.data, pt.nbytes, 0)
pt_ok = pt[:G, :n] > 0
pt = pt[:G, :n].astype(np.int64) - t0
kinds = ["qkv", "o", "gate_up_silu", "down"]
print(f"{'op':8s} {'span':>7s} {'wait1st':>8s} {'compute':>8s} {'flush':>7s} {'skewStart':>9s} {'skewDone':>8s}  (us, medians over layers)")
for k, name in enumerate(kinds):
    rows = []
    for j in range(k, n, len(kinds)):
        s, f1, l, d = b[:, j, 0], b[:, j, 1], b[:, j, 2], b[:, j, 3]
        rows.append([d.max() - s.min(), np.median(f1 - s), np.median(l - f1), np.median(d - l), s.max() - s.min(), d.max() - d.min()])
    r = np.median(np.array(rows), axis=0) / 1e3
    print(f"{name:8s} " + " ".join(f"{x:8.2f}" for x in r))
ends = [b[:, j, 3].max() for j in range(n)]
print("total span us:", (max(ends)) / 1e3)
# per-CTA spread of the compute phase (first stage -> last stage) for each op kind, summed over layers
for k, name in enumerate(kinds):
    comp = np.zeros(G)
    for j in range(k, n, len(kinds)):
        comp += (b[:, j, 2] - b[:, j, 1]) / 1e3
    q = np.percentile(comp, [0, 10, 50, 90, 100])
    order = np.argsort(comp)
    print(f"{name:8s} compute per CTA (sum over layers) p0/10/50/90/100: " + " ".join(f"{x:7.1f}" for x in q),
          "| slowest CTAs", order[-6:].tolist(), "| fastest", order[:6].tolist())

# last-segment flush decomposition: owner wait (slots 4 -> 5) and flush end (slot 6) vs loop end (slot 2)
for k, name in enumerate(kinds):
    ow, fl, dn = [], [], []
    for j in range(k, n, len(kinds)):
        w = b[:, j, 5] - b[:, j, 4]
        own = (buf[:G, j, 4] > 0) & (buf[:G, j, 5] >= buf[:G, j, 4])
        if own.any():
            ow.append(np.median(w[own]) / 1e3)
        fl.append(np.median(b[:, j, 6] - b[:, j, 2]) / 1e3)
        dn.append(np.median(b[:, j, 3] - b[:, j, 6]) / 1e3)
    print(f"{name:8s} owner wait (median over owners) {np.median(ow) if ow else 0:6.2f} us | last flush {np.median(fl):6.2f} us | done-count {np.median(dn):6.2f} us")

# op start -> descriptor loaded (slot 7) vs -> first stage ready (slot 1)
for k, name in enumerate(kinds):
    d = [np.median(b[:, j, 7] - b[:, j, 0]) / 1e3 for j in range(k, n, len(kinds)) if (buf[:G, j, 7] > 0).all()]
    print(f"{name:8s} descriptor load {np.median(d) if d else float('nan'):6.2f} us")

# critical-path view: for each op, T_dep = the last CTA's done-count of the op its activations depend on
# (the previous op in this forward); per CTA: first stage ready - T_dep, compute, flush+count, done - T_dep
print("\nper op (layers 2..): percentiles p0/p50/p90/p100 over CTAs, us; T_dep = previous op's last done-count")
pq = lambda v: "/".join(f"{x:5.1f}" for x in np.percentile(v / 1e3, [0, 50, 90, 100]))
for k, name in enumerate(kinds):
    rows = {"ready-Tdep": [], "compute": [], "flush+cnt": [], "done-Tdep": []}
    for j in range(len(kinds) + k, n, len(kinds)):
        Tdep = b[:, j - 1, 3].max()
        rows["ready-Tdep"].append(b[:, j, 1] - Tdep)
        rows["compute"].append(b[:, j, 2] - b[:, j, 1])
        rows["flush+cnt"].append(b[:, j, 3] - b[:, j, 2])
        rows["done-Tdep"].append(b[:, j, 3] - Tdep)
    print(f"{name:8s} " + "  ".join(f"{key} {pq(np.concatenate(v))}" for key, v in rows.items()))

# producer: activation load of the op's first stage issued (after its tile dependencies) vs consumers' first
# stage ready: the activation TMA's latency behind the weight stream
print("\nfirst stage of each op (layers 2..), p10/p50/p90 over CTAs, us: act issue - T_dep, ready - act issue")
for k, name in enumerate(kinds):
    a1, a2 = [], []
    for l in range(1, n // 4):
        j = 4 * l + k
        Tdep = b[:, j - 1, 3].max()
        ok = pt_ok[:, j]
        a1 += list((pt[ok, j] - Tdep) / 1e3)
        a2 += list((b[ok, j, 1] - pt[ok, j]) / 1e3)
    q = lambda v: "/".join(f"{x:5.2f}" for x in np.percentile(v, [10, 50, 90])) if v else "-"
    print(f"{name:12s} issue-Tdep {q(a1)}   ready-issue {q(a2)}")

# compute time vs the CTA's number of tile segments in the op (stream-K ranges of (K, N, G) only)
print("\ncompute per op (us, median over layers 2..) by the CTA's tile segments in the op")
shapes = {"qkv": (8192, 10240), "o": (8192, 8192), "gate_up_silu": (8192, 57344), "down": (28672, 8192)}
for k, name in enumerate(kinds):
    K, N = shapes[name]
    Gk, U = K // 128, (N // 128) * (K // 128)
    ub = [(c * U) // G for c in range(G + 1)]
    nseg = np.array([len({u // Gk for u in (ub[c], ub[c + 1] - 1)}) if ub[c + 1] - 1 - ub[c] < Gk else
                     (ub[c + 1] - 1) // Gk - ub[c] // Gk + 1 for c in range(G)])
    comp = np.median(np.stack([(b[:, j, 2] - b[:, j, 1]) / 1e3 for j in range(4 + k, n, 4)]), axis=0)
    out = []
    for sgs in sorted(set(nseg.tolist())):
        sel = nseg == sgs
        out.append(f"{sgs} seg: n={sel.sum():3d} median {np.median(comp[sel]):6.2f} p90 {np.percentile(comp[sel], 90):6.2f}")
    print(f"{name:12s} " + " | ".join(out))
