"""Seeded synthetic inputs shared by the oracle side and the GPU side (see synth.h).

Holds none of the method's arithmetic: weights/activations come from a counter-based generator with a
host (C) and a device (CUDA) implementation that produce bit-identical fp16; draft trees and target
argmax vectors come from numpy generators below (random numbers the method would draw are passed in).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
WEIGHT, ACT = 0, 1

_host = None
_gpu = None


def _host_lib():
    global _host
    if _host is None:
        so = os.path.join(_HERE, "libsynth_host.so")
        src = os.path.join(_HERE, "synth.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            import subprocess
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-o", so, src])
        _host = ctypes.CDLL(so)
        _host.synth_fill_host.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p]
        _host.synth_fill_host.restype = ctypes.c_int
        _host.synth_fill_host_block.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int] + [ctypes.c_int] * 6 + [
            ctypes.c_void_p]
        _host.synth_fill_host_block.restype = ctypes.c_int
        _host.synth_value_host.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int]
        _host.synth_value_host.restype = ctypes.c_uint16
    return _host


def _gpu_lib():
    global _gpu
    if _gpu is None:
        so = os.path.join(_HERE, "libsynth_gpu.so")
        if not os.path.exists(so):
            raise ImportError(f"{so} not built: run `make`")
        _gpu = ctypes.CDLL(so)
        _gpu.synth_fill_gpu.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p]
        _gpu.synth_fill_gpu.restype = ctypes.c_int
    return _gpu


def host(seed: int, tensor_id: int, kind: int, rows: int, cols: int) -> np.ndarray:
    """fp16 bit patterns (uint16) [rows, cols]."""
    out = np.empty((rows, cols), dtype=np.uint16)
    if _host_lib().synth_fill_host(seed, tensor_id, kind, rows, cols, out.ctypes.data) != 0:
        raise ValueError("synth_fill_host: bad arguments")
    return out


def host_block(seed, tensor_id, kind, rows, cols, r0, r1, c0, c1) -> np.ndarray:
    """Sub-block [r0:r1, c0:c1] of host(seed, tensor_id, kind, rows, cols), without generating the rest."""
    out = np.empty((r1 - r0, c1 - c0), dtype=np.uint16)
    if _host_lib().synth_fill_host_block(seed, tensor_id, kind, rows, cols, r0, r1, c0, c1, out.ctypes.data) != 0:
        raise ValueError("synth_fill_host_block: bad arguments")
    return out


def host_value(seed, tensor_id, kind, rows, cols, r, c) -> int:
    return int(_host_lib().synth_value_host(seed, tensor_id, kind, rows, cols, r, c))


def gpu(seed: int, tensor_id: int, kind: int, rows: int, cols: int, device=None, out=None):
    """torch.float16 CUDA tensor [rows, cols], bit-identical to host()."""
    import torch
    if out is None:
        out = torch.empty((rows, cols), dtype=torch.float16, device=device or "cuda")
    stream = torch.cuda.current_stream(out.device).cuda_stream
    if _gpu_lib().synth_fill_gpu(seed, tensor_id, kind, rows, cols, out.data_ptr(), stream) != 0:
        raise RuntimeError("synth_fill_gpu failed")
    return out


def tensor_id(layer: int, matrix: int, shard: int = 0) -> int:
    """Distinct generator stream per (layer, matrix, shard)."""
    return (layer << 16) | (matrix << 8) | shard


# ----------------------------------------------------------------------------------------------------
# Draft trees (EAGLE-2-shaped, depth <= d, top-k per expansion, top-n by cumulative
# log-prob) and target argmax vectors with a chosen per-edge acceptance rate.
# ----------------------------------------------------------------------------------------------------
def eagle_tree(rng: np.random.Generator, n_draft: int, depth: int, topk: int = 10, vocab: int = 128256):
    """Returns (tokens, parents) of n_draft+1 nodes (node 0 = root), parents[i] < i, distinct sibling tokens.

    Synthetic drafter: each expansion draws a Dirichlet-like distribution over topk fresh tokens; the tree keeps
    the n_draft highest cumulative log-prob nodes (parent-closed, since children score below parents)."""
    cand = [(0.0, -1, 0)]  # (logp, parent_index_in_nodes, depth)
    nodes = [(0.0, -1, 0, int(rng.integers(vocab)))]
    frontier = [0]
    for d in range(1, depth + 1):
        new = []
        for f in frontier:
            probs = np.sort(rng.dirichlet(np.full(topk, 0.3)))[::-1]
            toks = rng.choice(vocab, size=topk, replace=False)
            for p, t in zip(probs, toks):
                new.append((nodes[f][0] + float(np.log(max(p, 1e-12))), f, d, int(t)))
        new.sort(key=lambda x: -x[0])
        keep = new[:topk]
        base = len(nodes)
        nodes.extend(keep)
        frontier = list(range(base, base + len(keep)))
    # select top n_draft non-root nodes by score, parent-closed (scores decrease along paths)
    order = sorted(range(1, len(nodes)), key=lambda i: (-nodes[i][0], nodes[i][2], i))
    chosen = set()
    for i in order:
        if len(chosen) >= n_draft:
            break
        chain, x = [], i
        while x != 0 and x not in chosen:
            chain.append(x)
            x = nodes[x][1]
        if len(chosen) + len(chain) <= n_draft:
            chosen.update(chain)
    sel = sorted(chosen, key=lambda i: (nodes[i][2], i))  # BFS order => parent precedes child
    remap = {0: 0}
    for j, i in enumerate(sel, start=1):
        remap[i] = j
    tokens = [nodes[0][3]] + [nodes[i][3] for i in sel]
    parents = [-1] + [remap[nodes[i][1]] for i in sel]
    return np.array(tokens, dtype=np.int32), np.array(parents, dtype=np.int32)


def target_argmax_for(rng, tokens, parents, p_accept: float, vocab: int = 128256):
    """argmax[i] = token of one of i's children with prob p_accept (first child by index), else a token
    matching none of i's children."""
    n = len(tokens)
    children = [[] for _ in range(n)]
    for i in range(1, n):
        children[parents[i]].append(i)
    out = np.empty(n, dtype=np.int32)
    for i in range(n):
        ch_tokens = {int(tokens[c]) for c in children[i]}
        if children[i] and rng.random() < p_accept:
            out[i] = tokens[children[i][0]]
        else:
            t = int(rng.integers(vocab))
            while t in ch_tokens:
                t = int(rng.integers(vocab))
            out[i] = t
    return out
