#!/usr/bin/env python
"""Diagnostics: per-GEMM time of several (shape, M, family) combinations, each back to back over R distinct
weight copies in a CUDA graph (weights >> L2), CUDA events; one JSON line per combination.
  python tools/probe_fam.py --shapes gate_up,qkv --M 1,8,16,64 --families 0,1,3"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22179_b200 as w4
import synth

SHAPES = {"qkv": (8192, 10240), "o": (8192, 8192), "gate_up": (8192, 57344), "down": (28672, 8192), "c1": (4096, 4096)}
ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="gate_up")
ap.add_argument("--M", default="8")
ap.add_argument("--families", default="0,3")
ap.add_argument("--bytes", type=float, default=2.0e9, help="distinct weight bytes per graph (>> L2)")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6542.7
s = torch.cuda.Stream()
for name in a.shapes.split(","):
    K, N = SHAPES[name]
    wb = w4.w4a16_packed_bytes(K, N)
    R = max(2, int(a.bytes // wb))
    lins = []
    for r in range(R):
        W = synth.gpu(0, 100 + r, synth.WEIGHT, K, N)
        lins.append(w4.pack_linear(W)); del W
    torch.cuda.synchronize()
    for M in [int(m) for m in a.M.split(",")]:
        X = synth.gpu(0, 2, synth.ACT, M, K)
        Y = torch.empty(M, N, dtype=torch.float16, device="cuda")
        ws = w4.alloc_workspace(M, [(K, N)])
        for fam in [int(f) for f in a.families.split(",")]:
            if fam in (0, 2) and M > 16:
                continue
            try:
                with torch.cuda.stream(s):
                    for l in lins: l(X, Y, ws, s, family=fam)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for l in lins: l(X, Y, ws, s, family=fam)
                for _ in range(2): g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                with torch.cuda.stream(s):
                    for _ in range(a.reps): g.replay()
                e1.record(s)
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / (a.reps * R)
                print(json.dumps({"shape": name, "K": K, "N": N, "M": M, "family": fam, "us": round(us, 2),
                                  "GBps": round(wb / us / 1e3, 1), "frac": round(wb / us / 1e3 / peak, 3), "R": R}), flush=True)
                del g
            except Exception as e:
                print(json.dumps({"shape": name, "M": M, "family": fam, "error": repr(e)}), flush=True)
    del lins
    torch.cuda.empty_cache()

if int(os.environ.get("W4A16_TP_DEBUG", "0")) & 256:
    # per-unit timeline of CTA 0 of the last launch (gemm_tp.cu g_tp_trace), ns relative to the first event
    import ctypes
    import numpy as np
    from paper_2505_22179_b200._lib import lib
    buf = np.zeros((12, 128), dtype=np.uint64)
    lib.w4a16_debug_trace_tp(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    names = ["X_issue", "W_issue", "D0_wfull", "D1_wfull", "D_aempty", "M_ready", "M_commit", "D_afull", "E_accfull", "E_done"]
    t0 = int(buf[buf > 0].min()) if (buf > 0).any() else 0
    print("unit " + " ".join(f"{n:>10}" for n in names))
    for i in range(0, 64):
        print(f"{i:4d} " + " ".join(f"{(int(buf[e, i]) - t0) if buf[e, i] else -1:10d}" for e in range(len(names))))
