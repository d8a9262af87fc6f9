"""ctypes binding of the CPU oracle (oracle/w4a16_oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
package. The product (paper_2505_22179_b200/) never imports it, and the two share no code.
Arrays are numpy: fp16 tensors as uint16 bit patterns (or np.float16 views), qweight as uint32.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libw4a16_oracle.so")

ASYM, SYM = 0, 1
DEV_OK, DEV_NONFINITE, DEV_BAD_TREE = 0, 1, 2


def _build():
    src = os.path.join(_HERE, "w4a16_oracle.c")
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-o", _SO, src,
                           "-lm", "-lpthread"])


def _load():
    src = os.path.join(_HERE, "w4a16_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        _build()
    L = ctypes.CDLL(_SO)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.orc_half_to_float.argtypes = [ctypes.c_uint16]; L.orc_half_to_float.restype = ctypes.c_float
    L.orc_half_to_double.argtypes = [ctypes.c_uint16]; L.orc_half_to_double.restype = ctypes.c_double
    L.orc_float_to_half.argtypes = [ctypes.c_float]; L.orc_float_to_half.restype = ctypes.c_uint16
    L.orc_double_to_half.argtypes = [ctypes.c_double]; L.orc_double_to_half.restype = ctypes.c_uint16
    L.orc_quantize.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp, vp]; L.orc_quantize.restype = i32
    L.orc_dequantize.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp]; L.orc_dequantize.restype = i32
    L.orc_gemm.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, i32]; L.orc_gemm.restype = i32
    L.orc_gemm_cols.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, i32, vp]; L.orc_gemm_cols.restype = i32
    L.orc_gemm_exact.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, i32]; L.orc_gemm_exact.restype = i32
    L.orc_packed_bytes.argtypes = [i32, i32, i32]; L.orc_packed_bytes.restype = sz
    L.orc_code_word_offset.argtypes = [i32, i32, i32, i32, i32]; L.orc_code_word_offset.restype = sz
    L.orc_nibble_slot.argtypes = [i32]; L.orc_nibble_slot.restype = i32
    L.orc_layout_pack.argtypes = [vp, vp, vp, i32, i32, i32, vp]; L.orc_layout_pack.restype = i32
    L.orc_layout_unpack.argtypes = [vp, i32, i32, i32, vp, vp, vp]; L.orc_layout_unpack.restype = i32
    L.orc_accept.argtypes = [vp, vp, vp, i32, vp]; L.orc_accept.restype = i32
    L.orc_tree_attention.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp]; L.orc_tree_attention.restype = i32
    L.orc_kv_compact.argtypes = [vp, vp, i32, i32, i32, vp]; L.orc_kv_compact.restype = i32
    L.orc_hadamard.argtypes = [vp, i32, i32, i32, vp]; L.orc_hadamard.restype = i32
    L.orc_allreduce.argtypes = [vp, i32, ctypes.c_size_t, vp]; L.orc_allreduce.restype = i32
    L.orc_quantize_act_int8.argtypes = [vp, i32, i32, vp, vp, vp]; L.orc_quantize_act_int8.restype = i32
    L.orc_gemm_w4a8.argtypes = [vp, vp, vp, vp, i32, i32, i32, vp]; L.orc_gemm_w4a8.restype = i32
    L.orc_lmhead_argmax.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp, i32]; L.orc_lmhead_argmax.restype = i32
    return L


L = _load()


def _p(a):
    return None if a is None else a.ctypes.data


def _u16(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint16) if a.dtype == np.float16 else a.astype(np.uint16, copy=False)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def half_to_float(h: int) -> float:
    return L.orc_half_to_float(int(h))


def float_to_half(f: float) -> int:
    return L.orc_float_to_half(float(f))


def double_to_half(d: float) -> int:
    return L.orc_double_to_half(float(d))


def quantize(W, group=128, mode=ASYM):
    """W [K, N] fp16 -> (codes uint8 [K, N], scales uint16 [K/g, N], zeros uint16 [K/g, N] or None, status)."""
    W = _u16(W)
    K, N = W.shape
    codes = np.zeros((K, N), dtype=np.uint8)
    sc = np.zeros((K // group, N), dtype=np.uint16)
    ze = np.zeros((K // group, N), dtype=np.uint16) if mode == ASYM else None
    st = np.zeros(1, dtype=np.int32)
    if L.orc_quantize(_p(W), K, N, group, mode, _p(codes), _p(sc), _p(ze), _p(st)) != 0:
        raise ValueError("orc_quantize: bad arguments")
    return codes, sc, ze, int(st[0])


def dequantize(codes, sc, ze, group=128, mode=ASYM):
    codes = _c(codes, np.uint8)
    K, N = codes.shape
    out = np.zeros((K, N), dtype=np.uint16)
    if L.orc_dequantize(_p(codes), _p(_u16(sc)), _p(None if ze is None else _u16(ze)), K, N, group, mode, _p(out)) != 0:
        raise ValueError("orc_dequantize: bad arguments")
    return out


def gemm(X, codes, sc, ze, group=128, mode=ASYM, nthreads=1):
    """fp64 Y[M, N] = X[M, K] (fp16) . W_hat."""
    X = _u16(X)
    codes = _c(codes, np.uint8)
    K, N = codes.shape
    M = X.shape[0]
    Y = np.zeros((M, N), dtype=np.float64)
    if L.orc_gemm(_p(X), _p(codes), _p(_u16(sc)), _p(None if ze is None else _u16(ze)), M, K, N, group, mode, _p(Y),
                  int(nthreads)) != 0:
        raise ValueError("orc_gemm: bad arguments")
    return Y


def gemm_exact(X, codes, sc, ze, group=128, mode=ASYM, nthreads=1):
    """fp64 Y[M, N] = X . W with W = (q - z) * s exactly, no fp16 rounding of the weight (reading R22)."""
    X = _u16(X)
    codes = _c(codes, np.uint8)
    K, N = codes.shape
    M = X.shape[0]
    Y = np.zeros((M, N), dtype=np.float64)
    if L.orc_gemm_exact(_p(X), _p(codes), _p(_u16(sc)), _p(None if ze is None else _u16(ze)), M, K, N, group, mode,
                        _p(Y), int(nthreads)) != 0:
        raise ValueError("orc_gemm_exact: bad arguments")
    return Y


def gemm_cols(X, codes, sc, ze, cols, group=128, mode=ASYM):
    X = _u16(X)
    codes = _c(codes, np.uint8)
    K, N = codes.shape
    M = X.shape[0]
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    Y = np.zeros((M, cols.size), dtype=np.float64)
    if L.orc_gemm_cols(_p(X), _p(codes), _p(_u16(sc)), _p(None if ze is None else _u16(ze)), M, K, N, group, mode,
                       _p(cols), cols.size, _p(Y)) != 0:
        raise ValueError("orc_gemm_cols: bad arguments")
    return Y


def packed_bytes(K, N, mode=ASYM) -> int:
    return int(L.orc_packed_bytes(K, N, mode))


def code_word_offset(K, N, k, n, mode=ASYM) -> int:
    return int(L.orc_code_word_offset(K, N, mode, k, n))


def nibble_slot(i) -> int:
    return L.orc_nibble_slot(i)


def layout_pack(codes, sc, ze, mode=ASYM):
    codes = _c(codes, np.uint8)
    K, N = codes.shape
    out = np.zeros(packed_bytes(K, N, mode), dtype=np.uint8)
    if L.orc_layout_pack(_p(codes), _p(_u16(sc)), _p(None if ze is None else _u16(ze)), K, N, mode, _p(out)) != 0:
        raise ValueError("orc_layout_pack: bad arguments")
    return out


def layout_unpack(packed, K, N, mode=ASYM):
    packed = _c(packed, np.uint8)
    codes = np.zeros((K, N), dtype=np.uint8)
    sc = np.zeros((K // 128, N), dtype=np.uint16)
    ze = np.zeros((K // 128, N), dtype=np.uint16)
    if L.orc_layout_unpack(_p(packed), K, N, mode, _p(codes), _p(sc), _p(ze)) != 0:
        raise ValueError("orc_layout_unpack: bad arguments")
    return codes, sc, (ze if mode == ASYM else None)


def pack(W, mode=ASYM):
    """group-128 quantise + ABI byte layout: -> (packed uint8, codes, scales, zeros, status)."""
    codes, sc, ze, st = quantize(W, 128, mode)
    return layout_pack(codes, sc, ze, mode), codes, sc, ze, st


def accept(tokens, parents, argmax):
    """-> (accepted_len, bonus, status, path list)."""
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    p = np.ascontiguousarray(parents, dtype=np.int32)
    a = np.ascontiguousarray(argmax, dtype=np.int32)
    n = t.size
    out = np.zeros(3 + n, dtype=np.int32)
    rc = L.orc_accept(_p(t), _p(p), _p(a), n, _p(out))
    if rc != 0:
        raise ValueError("orc_accept: bad arguments")
    return int(out[0]), int(out[1]), int(out[2]), [int(x) for x in out[3:3 + out[0]]], out


def lmhead_argmax(H, W, nthreads=1, want_logits=False):
    """Greedy token per row: (argmax int32 [M], max logit fp64 [M][, logits fp64 [M][V]]) of H[M,K] . W[V,K]^T
    (fp16 inputs, fp64 logits, ties -> lowest id)."""
    H, W = _u16(H), _u16(W)
    M, K = H.shape
    V = W.shape[0]
    if W.shape[1] != K:
        raise ValueError("lmhead_argmax: K mismatch")
    idx = np.zeros(M, dtype=np.int32)
    val = np.zeros(M, dtype=np.float64)
    lg = np.zeros((M, V), dtype=np.float64) if want_logits else None
    if L.orc_lmhead_argmax(_p(H), _p(W), M, K, V, _p(idx), _p(val), _p(lg), int(nthreads)) != 0:
        raise ValueError("orc_lmhead_argmax: bad arguments")
    return (idx, val, lg) if want_logits else (idx, val)


def tree_attention(Q, Kc, Vc, parents):
    """fp64 O[M, Hq, D] of the tree-masked verify attention. Q fp16 [M, Hq, D]; Kc, Vc fp16
    [L + M, Hkv, D]; parents int32 [M]."""
    Q, Kc, Vc = _u16(Q), _u16(Kc), _u16(Vc)
    M, Hq, D = Q.shape
    Lt, Hkv, D2 = Kc.shape
    if D2 != D or Vc.shape != Kc.shape or Lt < M:
        raise ValueError("tree_attention: shapes")
    par = np.ascontiguousarray(parents, dtype=np.int32)
    O = np.zeros((M, Hq, D), dtype=np.float64)
    if L.orc_tree_attention(_p(Q), _p(Kc), _p(Vc), _p(par), M, Lt - M, Hq, Hkv, D, _p(O)) != 0:
        raise ValueError("orc_tree_attention: bad arguments")
    return O


def kv_compact(Kc, Vc, L_prefix, accept_out):
    """In-place on copies: returns (Kc', Vc') (input dtype) with the accepted path's rows moved behind the root."""
    dt = np.asarray(Kc).dtype
    Kc = _u16(Kc).copy()
    Vc = _u16(Vc).copy()
    Lt, Hkv, D = Kc.shape
    out = np.ascontiguousarray(accept_out, dtype=np.int32)
    if L.orc_kv_compact(_p(Kc), _p(Vc), int(L_prefix), Hkv, D, _p(out)) != 0:
        raise ValueError("orc_kv_compact: bad arguments")
    return (Kc.view(np.float16), Vc.view(np.float16)) if dt == np.float16 else (Kc, Vc)


def hadamard(X, B=128):
    """fp64 block Hadamard rotation along the last axis: X fp16 [M, K] -> fp64 [M, K]."""
    X = _u16(X)
    M, K = X.shape
    Y = np.zeros((M, K), dtype=np.float64)
    if L.orc_hadamard(_p(X), M, K, int(B), _p(Y)) != 0:
        raise ValueError("orc_hadamard: bad arguments")
    return Y


def allreduce(P):
    """Sum over tensor-parallel ranks: P fp16 [T, ...] -> fp16 [...], fp64 sum rounded once."""
    P = _u16(P)
    T = P.shape[0]
    out = np.zeros(P.shape[1:], dtype=np.uint16)
    if L.orc_allreduce(_p(P), T, out.size, _p(out)) != 0:
        raise ValueError("orc_allreduce: bad arguments")
    return out


def quantize_act_int8(X):
    """W4A8 activations (reading R21): fp16 [M, K] -> (Xq int8 [M, K], sx fp32 [M], xsum int32 [M, K/128])."""
    X = _u16(X)
    M, K = X.shape
    Xq = np.zeros((M, K), dtype=np.int8)
    sx = np.zeros(M, dtype=np.float32)
    xs = np.zeros((M, K // 128), dtype=np.int32)
    if L.orc_quantize_act_int8(_p(X), M, K, _p(Xq), _p(sx), _p(xs)) != 0:
        raise ValueError("orc_quantize_act_int8: bad arguments")
    return Xq, sx, xs


def gemm_w4a8(Xq, sx, codes, sc):
    """W4A8 GEMM on SYM g128 weights (codes uint8 [K, N], scales fp16 bits [K/128, N]) -> fp64 [M, N]."""
    Xq = np.ascontiguousarray(Xq, dtype=np.int8)
    sx = np.ascontiguousarray(sx, dtype=np.float32)
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    sc = _u16(sc)
    M, K = Xq.shape
    N = codes.shape[1]
    Y = np.zeros((M, N), dtype=np.float64)
    if L.orc_gemm_w4a8(_p(Xq), _p(sx), _p(codes), _p(sc), M, K, N, _p(Y)) != 0:
        raise ValueError("orc_gemm_w4a8: bad arguments")
    return Y
