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
    vp, i32 = ctypes.c_void_p, ctypes.c_int
    L.orc_half_to_float.argtypes = [ctypes.c_uint16]; L.orc_half_to_float.restype = ctypes.c_float
    L.orc_half_to_double.argtypes = [ctypes.c_uint16]; L.orc_half_to_double.restype = ctypes.c_double
    L.orc_float_to_half.argtypes = [ctypes.c_float]; L.orc_float_to_half.restype = ctypes.c_uint16
    L.orc_double_to_half.argtypes = [ctypes.c_double]; L.orc_double_to_half.restype = ctypes.c_uint16
    L.orc_word_index.argtypes = [i32, i32, i32, i32]; L.orc_word_index.restype = ctypes.c_size_t
    L.orc_nibble_slot.argtypes = [i32]; L.orc_nibble_slot.restype = i32
    L.orc_get_code.argtypes = [vp, i32, i32, i32, i32]; L.orc_get_code.restype = i32
    L.orc_pack.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp, vp]; L.orc_pack.restype = i32
    L.orc_unpack.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp]; L.orc_unpack.restype = i32
    L.orc_gemm.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, i32]; L.orc_gemm.restype = i32
    L.orc_gemm_cols.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, i32, vp]; L.orc_gemm_cols.restype = i32
    L.orc_accept.argtypes = [vp, vp, vp, i32, vp]; L.orc_accept.restype = i32
    return L


L = _load()


def _p(a):
    return None if a is None else a.ctypes.data


def _u16(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint16) if a.dtype == np.float16 else a.astype(np.uint16, copy=False)


def half_to_float(h: int) -> float:
    return L.orc_half_to_float(int(h))


def float_to_half(f: float) -> int:
    return L.orc_float_to_half(float(f))


def double_to_half(d: float) -> int:
    return L.orc_double_to_half(float(d))


def pack(W, group=128, mode=ASYM):
    """W: [K, N] fp16 -> (qweight uint32 [K*N/8], scales uint16 [K/g, N], zeros uint16 or None, status)."""
    W = _u16(W)
    K, N = W.shape
    qw = np.zeros(K * N // 8, dtype=np.uint32)
    sc = np.zeros((K // group, N), dtype=np.uint16)
    ze = np.zeros((K // group, N), dtype=np.uint16) if mode == ASYM else None
    st = np.zeros(1, dtype=np.int32)
    rc = L.orc_pack(_p(W), K, N, group, mode, _p(qw), _p(sc), _p(ze), _p(st))
    if rc != 0:
        raise ValueError("orc_pack: bad arguments")
    return qw, sc, ze, int(st[0])


def unpack(qw, sc, ze, K, N, group=128, mode=ASYM):
    out = np.zeros((K, N), dtype=np.uint16)
    rc = L.orc_unpack(_p(np.ascontiguousarray(qw, dtype=np.uint32)), _p(_u16(sc)), _p(None if ze is None else _u16(ze)),
                      K, N, group, mode, _p(out))
    if rc != 0:
        raise ValueError("orc_unpack: bad arguments")
    return out


def gemm(X, qw, sc, ze, K, N, group=128, mode=ASYM, nthreads=1):
    """fp64 Y[M, N] = X[M, K] (fp16) . W_hat."""
    X = _u16(X)
    M = X.shape[0]
    Y = np.zeros((M, N), dtype=np.float64)
    rc = L.orc_gemm(_p(X), _p(np.ascontiguousarray(qw, dtype=np.uint32)), _p(_u16(sc)),
                    _p(None if ze is None else _u16(ze)), M, K, N, group, mode, _p(Y), int(nthreads))
    if rc != 0:
        raise ValueError("orc_gemm: bad arguments")
    return Y


def gemm_cols(X, qw, sc, ze, K, N, cols, group=128, mode=ASYM):
    X = _u16(X)
    M = X.shape[0]
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    Y = np.zeros((M, cols.size), dtype=np.float64)
    rc = L.orc_gemm_cols(_p(X), _p(np.ascontiguousarray(qw, dtype=np.uint32)), _p(_u16(sc)),
                         _p(None if ze is None else _u16(ze)), M, K, N, group, mode, _p(cols), cols.size, _p(Y))
    if rc != 0:
        raise ValueError("orc_gemm_cols: bad arguments")
    return Y


def get_code(qw, K, N, k, n) -> int:
    return L.orc_get_code(_p(np.ascontiguousarray(qw, dtype=np.uint32)), K, N, k, n)


def word_index(K, N, k, n) -> int:
    return L.orc_word_index(K, N, k, n)


def nibble_slot(i) -> int:
    return L.orc_nibble_slot(i)


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
