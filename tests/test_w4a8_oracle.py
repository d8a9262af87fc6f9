"""W4A8 oracle (PAPER P:105-106 QQQ-style symmetric W4A8; reading R21 in DESIGN.md) pinned to
facts that do not re-type its formulas: exactly representable activation grids, the row maximum, zero rows,
round-half-to-even ties, the quantisation error bound; the GEMM against numpy integer matmuls per group, a
closed form, and the fp64 W4A16 oracle within the activation-quantisation error bound."""
import numpy as np

import oracle

SYM = 1


def test_act_quant_exact_grid_and_row_max():
    A = 3.0
    j = np.arange(-127, 128, dtype=np.int64)
    ks = np.resize(j, 256)
    X = (ks * (A / 127.0)).astype(np.float16).reshape(1, 256)
    Xq, sx, xs = oracle.quantize_act_int8(X)
    # the grid survives fp16 rounding closely enough that every code is recovered exactly
    assert np.array_equal(Xq[0].astype(np.int64), ks)
    assert Xq[0].max() == 127 and Xq[0].min() == -127
    amax = np.abs(X.astype(np.float32)).max()
    assert sx[0] == np.float32(amax) / np.float32(127.0)
    assert np.array_equal(xs[0], [ks[:128].sum(), ks[128:].sum()])


def test_act_quant_zero_row_and_ties():
    X = np.zeros((2, 128), dtype=np.float16)
    X[1, 0] = 127.0          # inv = 1 exactly: q = rne(x)
    X[1, 1:6] = [0.5, 1.5, 2.5, -0.5, -2.5]
    Xq, sx, xs = oracle.quantize_act_int8(X)
    assert not Xq[0].any() and sx[0] == 0.0 and xs[0, 0] == 0
    assert list(Xq[1, :6]) == [127, 0, 2, 2, 0, -2]   # halves go to the even neighbour
    assert sx[1] == np.float32(1.0)


def test_act_quant_error_bound():
    rng = np.random.default_rng(3)
    X = (rng.standard_normal((8, 1024)) * rng.choice([1e-3, 1.0, 40.0], size=(8, 1))).astype(np.float16)
    Xq, sx, xs = oracle.quantize_act_int8(X)
    x = X.astype(np.float64)
    err = np.abs(x - Xq.astype(np.float64) * sx[:, None].astype(np.float64))
    assert np.all(err <= sx[:, None] * (0.5 + 1e-5))
    assert np.array_equal(xs, Xq.astype(np.int32).reshape(8, -1, 128).sum(axis=2))


def test_w4a8_gemm_closed_form_and_numpy_per_group():
    rng = np.random.default_rng(4)
    M, K, N = 5, 384, 200
    Xq = rng.integers(-127, 128, size=(M, K)).astype(np.int8)
    sx = np.ones(M, dtype=np.float32)
    codes = np.full((K, N), 9, dtype=np.uint8)                 # q - 8 = 1
    sc = np.full((K // 128, N), np.float16(1.0)).view(np.uint16)
    Y = oracle.gemm_w4a8(Xq, sx, codes, sc)
    assert np.array_equal(Y, np.repeat(Xq.astype(np.int64).sum(axis=1, keepdims=True), N, axis=1).astype(np.float64))
    # general case: numpy integer matmul per group, then the scales (non-square: a transposed operand fails)
    codes = rng.integers(0, 16, size=(K, N)).astype(np.uint8)
    scf = (rng.uniform(0.5, 2.0, size=(K // 128, N))).astype(np.float16)
    sx = rng.uniform(0.01, 0.1, size=M).astype(np.float32)
    Y = oracle.gemm_w4a8(Xq, sx, codes, scf.view(np.uint16))
    ref = np.zeros((M, N))
    for g in range(K // 128):
        dot = Xq[:, g * 128:(g + 1) * 128].astype(np.int64) @ (codes[g * 128:(g + 1) * 128].astype(np.int64) - 8)
        ref += dot.astype(np.float64) * scf[g].astype(np.float64)[None, :]
    ref *= sx.astype(np.float64)[:, None]
    assert np.allclose(Y, ref, rtol=1e-12, atol=0)


def test_w4a8_close_to_w4a16_within_activation_quantisation_bound():
    rng = np.random.default_rng(5)
    M, K, N = 4, 512, 96
    W = (rng.standard_normal((K, N)) * 0.02).astype(np.float16)
    X = rng.standard_normal((M, K)).astype(np.float16)
    codes, sc, _, _ = oracle.quantize(W, 128, SYM)
    ref = oracle.gemm(X.view(np.uint16), codes, sc, None, mode=SYM)    # fp16 activations, same weights
    Xq, sx, _ = oracle.quantize_act_int8(X)
    Y = oracle.gemm_w4a8(Xq, sx, codes, sc)
    w_hat = (codes.astype(np.float64) - 8) * np.repeat(sc.view(np.float16).astype(np.float64), 128, axis=0)
    bound = (sx.astype(np.float64)[:, None] * 0.5 * 1.00001) @ np.abs(w_hat).sum(axis=0, keepdims=True) / 1.0
    assert np.all(np.abs(Y - ref) <= bound + 1e-9)
