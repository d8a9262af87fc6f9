"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a library routine (numpy), a closed form derived by hand,
a golden fixture (tests/golden/, with its citation), brute force on tiny inputs, or an invariant the
method must satisfy (losslessness vs autoregressive decoding). Chosen so that a dropped term, a wrong
sign/index, a transposed operand or a wrong nibble slot fails at least one of them.
"""
import itertools
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(1234)


# ---------------------------------------------------------------------------------------------------
# fp16 conversions (reading R1) — pinned to numpy's IEEE conversions (library routine).
# ---------------------------------------------------------------------------------------------------
def test_half_to_float_exhaustive():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([oracle.L.orc_half_to_double(int(b)) for b in bits])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])
    # and the float path agrees bit-for-bit (incl. signed zeros)
    sel = bits[::97]
    gotf = np.array([oracle.half_to_float(int(b)) for b in sel], dtype=np.float32)
    reff = sel.view(np.float16).astype(np.float32)
    ok = np.isnan(reff) & np.isnan(gotf)
    assert np.array_equal(gotf.view(np.uint32)[~ok], reff.view(np.uint32)[~ok])


def _edge_floats():
    e = [0.0, -0.0, 65504.0, 65519.99, 65520.0, 65536.0, -65520.0, 1e-8, 2.0 ** -24, 2.0 ** -25, 2.0 ** -25 * 1.0001,
         3 * 2.0 ** -26, 2.0 ** -14, 2.0 ** -14 - 2.0 ** -25, 6.1e-5, np.inf, -np.inf, 1.0 + 2.0 ** -11,
         1.0 + 3 * 2.0 ** -11, 1.0 + 2.0 ** -11 + 2.0 ** -30, 2049.0, 2051.0, 0.1, -0.1, 1.0 / 3.0]
    # all halfway points between consecutive representable halves in [1, 2) and in the subnormal range
    h = np.arange(0x3C00, 0x4000, 37, dtype=np.uint16).view(np.float16).astype(np.float64)
    e += list(h + 2.0 ** -11)
    s = np.arange(0, 1024, 13, dtype=np.uint16).view(np.float16).astype(np.float64)
    e += list(s + 2.0 ** -25)
    return np.array(e, dtype=np.float64)


def test_float_to_half_rne_vs_numpy():
    x = np.concatenate([_edge_floats(), RNG.standard_normal(100000) * 10.0 ** RNG.integers(-9, 5, 100000)])
    x32 = x.astype(np.float32)
    ref = x32.astype(np.float16).view(np.uint16)
    got = np.array([oracle.float_to_half(float(v)) for v in x32], dtype=np.uint16)
    assert np.array_equal(got, ref)


def test_double_to_half_rne_vs_numpy():
    x = np.concatenate([_edge_floats(), RNG.standard_normal(100000) * 10.0 ** RNG.integers(-9, 5, 100000)])
    ref = x.astype(np.float16).view(np.uint16)
    got = np.array([oracle.double_to_half(float(v)) for v in x], dtype=np.uint16)
    assert np.array_equal(got, ref)
    assert oracle.double_to_half(float("nan")) & 0x7C00 == 0x7C00


# ---------------------------------------------------------------------------------------------------
# Packed layout and nibble order — golden worked example (tests/golden/nibble_order.txt).
# ---------------------------------------------------------------------------------------------------
def hand_group(K, N):
    """w[k][n] = (((k+n) mod 16) - 4) * 2^-(3 + n mod 4): exactly representable with s_n = 2^-(3+n%4), z = 4,
    q = (k+n) mod 16 (derivation: wmin = -4 s, wmax = 11 s, (wmax-wmin)/15 = s exactly)."""
    k = np.arange(K)[:, None]
    n = np.arange(N)[None, :]
    w = (((k + n) % 16) - 4) * 2.0 ** (-(3 + n % 4))
    return w.astype(np.float16)


def _read_golden(name):
    rows = {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            rows.setdefault(key, []).append(vals)
    return rows


def test_nibble_order_golden():
    lines = [l.split() for l in open(os.path.join(GOLD, "nibble_order.txt")) if l.strip() and not l.startswith("#")]
    K = N = 128
    W = hand_group(K, N)  # column 0: q = k mod 16
    packed, codes_all, sc, ze, st = oracle.pack(W)
    for j, (codes, canon, phys) in enumerate(lines):
        codes = [int(c) for c in codes.split(",")]
        assert [int(codes_all[8 * j + i, 0]) for i in range(8)] == codes
        assert sum(c << (4 * i) for i, c in enumerate(codes)) == int(canon, 16)
        off = oracle.code_word_offset(K, N, 8 * j, 0)
        word = int.from_bytes(packed[off:off + 4].tobytes(), "little")
        assert word == int(phys, 16)
        # the LOP3 extraction the kernels use yields the consecutive-k pair in the two halves
        pair = word & 0x000F000F
        assert (pair & 0xFFFF, pair >> 16) == (codes[0], codes[1])
        pair = (word >> 8) & 0x000F000F
        assert (pair & 0xFFFF, pair >> 16) == (codes[4], codes[5])


@pytest.mark.parametrize("mode,TB", [(oracle.ASYM, 8704), (oracle.SYM, 8448)])
def test_layout_tiles_are_n_major_contiguous(mode, TB):
    K, N = 384, 256
    off = lambda k, n: oracle.code_word_offset(K, N, k, n, mode)  # noqa: E731
    assert off(0, 0) == 0 and off(8, 0) == 4 and off(0, 1) == 64
    assert off(32, 0) == 16 and off(32, 2) == 2 * 64 + 0 and off(0, 2) == 2 * 64 + 16   # chunk XOR (r/2)%4
    assert off(96, 7) == 7 * 64 + 16 * (3 ^ 3) and off(64, 5) == 5 * 64 + 16 * (2 ^ 2)
    assert off(128, 0) == TB                                  # next k-group, same n-tile
    assert off(0, 128) == 3 * TB                              # next n-tile after K/128 groups
    assert oracle.packed_bytes(K, N, mode) == 6 * TB
    # the 16-byte chunks a warp of 8 consecutive rows reads for one k-range hit 8 distinct bank groups
    for p4 in range(4):
        groups = {(off(32 * p4, r) % 128) // 16 for r in range(8)}
        assert len(groups) == 8
    # code words cover exactly the first 8192 bytes of every tile (a bijection)
    words = {off(k, n) for k in range(0, K, 8) for n in range(N)}
    expect = {t * TB + b for t in range(6) for b in range(0, 8192, 4)}
    assert words == expect


@pytest.mark.parametrize("mode", [oracle.ASYM, oracle.SYM])
def test_layout_scales_zeros_placement_and_roundtrip(mode):
    K, N = 256, 384
    W = synth.host(4, 5, synth.WEIGHT, K, N)
    codes, sc, ze, st = oracle.quantize(W, 128, mode)
    packed = oracle.layout_pack(codes, sc, ze, mode)
    TB = 8704 if mode == oracle.ASYM else 8448
    for g in range(K // 128):
        for n in (0, 1, 127, 128, 200, 383):
            t = (n // 128) * (K // 128) + g
            so = t * TB + 8192 + (4 if mode == oracle.ASYM else 2) * (n % 128)   # {s, z} side by side (ASYM)
            assert int.from_bytes(packed[so:so + 2].tobytes(), "little") == int(sc[g, n])
            if mode == oracle.ASYM:
                assert int.from_bytes(packed[so + 2:so + 4].tobytes(), "little") == int(ze[g, n])
    c2, s2, z2 = oracle.layout_unpack(packed, K, N, mode)
    assert np.array_equal(c2, codes) and np.array_equal(s2, sc)
    if mode == oracle.ASYM:
        assert np.array_equal(z2, ze)


# ---------------------------------------------------------------------------------------------------
# Pack / unpack — hand-computed group, SPEC example, degenerate groups, error bound.
# ---------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("K,N", [(128, 128), (256, 384)])
def test_pack_hand_group_exact_roundtrip(K, N):
    W = hand_group(K, N)
    codes, sc, ze, st = oracle.quantize(W)
    assert st == oracle.DEV_OK
    n = np.arange(N)
    assert np.array_equal(sc.view(np.float16).astype(np.float64), np.broadcast_to(2.0 ** (-(3 + n % 4)), sc.shape))
    assert np.all(ze.view(np.float16) == 4)
    k = np.arange(K)[:, None]
    assert np.array_equal(codes, ((k + n[None, :]) % 16).astype(np.uint8))
    Wh = oracle.dequantize(codes, sc, ze)
    assert np.array_equal(Wh, W.view(np.uint16))


def test_pack_spec_example_sym():
    g = _read_golden("spec_sym_example.txt")
    w = [float(x) for x in g["w"][0]]
    K, N = 128, 128
    W = np.zeros((K, N), dtype=np.float16)
    W[:4, 0] = w
    codes, sc, ze, st = oracle.quantize(W, group=4, mode=oracle.SYM)
    assert int(sc[0, 0]) == int(g["scale_bits"][0][0], 16)
    assert [int(codes[k, 0]) for k in range(4)] == [int(c) for c in g["codes"][0]]
    Wh = oracle.dequantize(codes, sc, ze, group=4, mode=oracle.SYM).view(np.float16)
    assert [float(x) for x in Wh[:4, 0]] == [float(x) for x in g["w_hat"][0]]


def _f(vals):
    return [float(x) for x in vals]


def test_pack_rne_ties_golden_asym():
    # reading R4 (round half to even, GPTQ torch.round): exact ties of the zero point -wmin/s = 2.5 and of
    # the codes w/s = k + 0.5 (tests/golden/rne_ties.txt derives every value; half-away-from-zero fails it)
    g = _read_golden("rne_ties.txt")
    w = _f(g["asym_w"][0])
    W = np.zeros((128, 2), dtype=np.float16)
    W[: len(w), 1] = w
    codes, sc, ze, st = oracle.quantize(W, mode=oracle.ASYM)
    assert st == 0
    assert int(sc[0, 1]) == int(g["asym_scale"][0][0], 16)
    assert float(ze.view(np.float16)[0, 1]) == float(g["asym_zero"][0][0])
    assert [int(c) for c in codes[: len(w), 1]] == [int(c) for c in g["asym_codes"][0]]
    assert int(codes[len(w), 1]) == int(g["asym_codes"][0][-1])   # the padding zeros code to z
    Wh = oracle.dequantize(codes, sc, ze, mode=oracle.ASYM).view(np.float16)
    assert [float(x) for x in Wh[: len(w), 1]] == _f(g["asym_w_hat"][0])


def test_pack_rne_ties_golden_sym():
    g = _read_golden("rne_ties.txt")
    w = _f(g["sym_w"][0])
    W = np.zeros((128, 1), dtype=np.float16)
    W[: len(w), 0] = w
    codes, sc, ze, st = oracle.quantize(W, mode=oracle.SYM)
    assert int(sc[0, 0]) == int(g["sym_scale"][0][0], 16)
    assert [int(c) for c in codes[: len(w), 0]] == [int(c) for c in g["sym_codes"][0]]


def test_w4a8_act_rne_ties_golden():
    # reading R21: per-token int8 codes decided by RNE in fp32 (tests/golden/rne_ties.txt)
    g = _read_golden("rne_ties.txt")
    x = _f(g["act_x"][0])
    X = np.zeros((1, 128), dtype=np.float16)
    X[0, : len(x)] = x
    Xq, sx, xs = oracle.quantize_act_int8(X)
    assert float(sx[0]) == float(g["act_sx"][0][0])
    assert [int(v) for v in Xq[0, : len(x)]] == [int(v) for v in g["act_q"][0]]
    assert int(xs[0, 0]) == sum(int(v) for v in g["act_q"][0])


@pytest.mark.parametrize("mode", [oracle.ASYM, oracle.SYM])
def test_pack_all_zero_group(mode):
    # reading R15 (GPTQ): an all-zero group gets the range (-1, 1): s = fp16(2/15), q = z = 8, w_hat = 0
    W = np.zeros((128, 128), dtype=np.float16)
    codes, sc, ze, st = oracle.quantize(W, mode=mode)
    assert np.all(sc == 0x3044)
    assert np.all(codes == 8)
    if mode == oracle.ASYM:
        assert np.all(ze.view(np.float16) == 8)
    assert np.all(oracle.dequantize(codes, sc, ze, mode=mode) == 0)


def test_pack_nonfinite_flags_status_and_counts_as_zero():
    W = hand_group(128, 128)
    W2 = W.copy()
    W2[5, 3] = np.inf
    W2[6, 3] = np.nan
    qw, sc, ze, st = oracle.quantize(W2)
    assert st == oracle.DEV_NONFINITE
    W3 = W.copy()
    W3[5, 3] = 0
    W3[6, 3] = 0
    qw3, sc3, ze3, st3 = oracle.quantize(W3)
    assert st3 == oracle.DEV_OK
    assert np.array_equal(qw, qw3) and np.array_equal(sc, sc3) and np.array_equal(ze, ze3)


def test_pack_nonneg_group_zero_point_is_plus_zero():
    W = np.abs(hand_group(128, 128))
    qw, sc, ze, st = oracle.quantize(W)
    assert np.all(ze == 0)          # fp16 +0, never 0x8000


@pytest.mark.parametrize("mode", [oracle.ASYM, oracle.SYM])
def test_pack_error_bound_and_zero_exact(mode):
    # |w - w_hat| <= s/2 + 15*2^-11*s (fp16 rounding of s can force one clamp) + half an fp16 ulp of w_hat
    K, N = 512, 256
    W = synth.host(7, 3, synth.WEIGHT, K, N).view(np.float16)
    W[::17, ::13] = 0.0
    qw, sc, ze, st = oracle.quantize(W, mode=mode)
    Wh = oracle.dequantize(qw, sc, ze, mode=mode).view(np.float16).astype(np.float64)
    w = W.astype(np.float64)
    s = np.repeat(sc.view(np.float16).astype(np.float64), 128, axis=0)
    bound = s * (0.5 + 15 * 2.0 ** -11 + 1e-6) + np.abs(Wh) * 2.0 ** -11 + 2.0 ** -25
    assert np.all(np.abs(w - Wh) <= bound)
    assert np.all(Wh[w == 0] == 0)  # 0 is always representable (reading R3)
    # codes in range and zero points are integers in [0, 15]
    if mode == oracle.ASYM:
        z = ze.view(np.float16).astype(np.float64)
        assert np.all((z >= 0) & (z <= 15) & (z == np.round(z)))


def test_pack_sym_zero_is_eight_and_range_centered():
    K, N = 256, 128
    W = synth.host(3, 9, synth.WEIGHT, K, N)
    qw, sc, ze, st = oracle.quantize(W, mode=oracle.SYM)
    assert ze is None
    Wh = oracle.dequantize(qw, sc, None, mode=oracle.SYM).view(np.float16).astype(np.float64)
    s = sc.view(np.float16).astype(np.float64)
    # every dequantised value is an integer multiple of its scale in [-8, 7]
    r = Wh / np.repeat(s, 128, axis=0)
    # (w_hat is (q-8)*s rounded once to fp16: within 8 * 2^-11 of an integer multiple of s)
    assert np.all(np.abs(r - np.round(r)) <= 8 * 2.0 ** -11) and np.round(r).min() >= -8 and np.round(r).max() <= 7


# ---------------------------------------------------------------------------------------------------
# GEMM reference — closed forms, one-hot exactness, numpy float64 matmul.
# ---------------------------------------------------------------------------------------------------
def test_gemm_ones_closed_form():
    # X = ones, hand group, K = 4096: Y[n] = s_n * sum_k ((k+n)%16 - 4) = s_n * 256 * (120 - 64) = 14336 s_n
    K, N = 4096, 256
    W = hand_group(K, N)
    qw, sc, ze, st = oracle.quantize(W)
    X = np.ones((2, K), dtype=np.float16)
    Y = oracle.gemm(X, qw, sc, ze, nthreads=4)
    n = np.arange(N)
    exp = 14336.0 * 2.0 ** (-(3 + n % 4))
    assert np.array_equal(Y[0], exp) and np.array_equal(Y[1], exp)
    assert list(exp[:4]) == [1792.0, 896.0, 448.0, 224.0]


def test_gemm_one_hot_rows_select_dequantised_weights():
    K, N = 512, 256
    W = synth.host(5, 1, synth.WEIGHT, K, N)
    qw, sc, ze, st = oracle.quantize(W)
    Wh = oracle.dequantize(qw, sc, ze).view(np.float16).astype(np.float64)
    ks = [0, 1, 7, 8, 127, 128, 300, 511]
    X = np.zeros((len(ks), K), dtype=np.float16)
    for m, k in enumerate(ks):
        X[m, k] = 1.0
    Y = oracle.gemm(X, qw, sc, ze)
    assert np.array_equal(Y, Wh[ks])


@pytest.mark.parametrize("mode", [oracle.ASYM, oracle.SYM])
def test_gemm_matches_numpy_float64(mode):
    K, N, M = 640, 384, 5
    W = synth.host(11, 2, synth.WEIGHT, K, N)
    X = synth.host(11, 3, synth.ACT, M, K)
    qw, sc, ze, st = oracle.quantize(W, mode=mode)
    Wh = oracle.dequantize(qw, sc, ze, mode=mode).view(np.float16).astype(np.float64)
    ref = X.view(np.float16).astype(np.float64) @ Wh
    Y1 = oracle.gemm(X, qw, sc, ze, mode=mode, nthreads=1)
    Y3 = oracle.gemm(X, qw, sc, ze, mode=mode, nthreads=3)
    assert np.array_equal(Y1, Y3)                          # thread count never changes the result
    assert np.allclose(Y1, ref, rtol=1e-12, atol=1e-12)
    cols = np.array([0, 5, 127, 128, 383])
    assert np.array_equal(oracle.gemm_cols(X, qw, sc, ze, cols, mode=mode), Y1[:, cols])


@pytest.mark.parametrize("mode", [oracle.ASYM, oracle.SYM])
def test_gemm_exact_weights_pins(mode):
    # reading R22: orc_gemm_exact uses the exact quantised weight (q - z) * s. Pinned to (i) one-hot rows = the
    # exact products (a 4-bit integer times an fp16 scale, exact in double), whose fp16 rounding is the
    # dequantised weight of orc_dequantize (consistency of the two definitions); (ii) a numpy float64 matmul of
    # (codes - z) * s built from the codes (library routine); (iii) the definitional gap to orc_gemm is bounded
    # by sum_k |x_k| ulp16(w_hat_k) / 2
    K, N, M = 640, 384, 5
    W = synth.host(13, 2, synth.WEIGHT, K, N)
    X = synth.host(13, 3, synth.ACT, M, K)
    qw, sc, ze, st = oracle.quantize(W, mode=mode)
    z = np.full((K // 128, N), 8.0) if mode == oracle.SYM else ze.view(np.float16).astype(np.float64)
    s = sc.view(np.float16).astype(np.float64)
    Wx = (qw.astype(np.float64) - np.repeat(z, 128, axis=0)) * np.repeat(s, 128, axis=0)
    ks = [0, 1, 7, 127, 128, 300, 639]
    Xh = np.zeros((len(ks), K), dtype=np.float16)
    for m, k in enumerate(ks):
        Xh[m, k] = 1.0
    Yh = oracle.gemm_exact(Xh, qw, sc, ze, mode=mode)
    assert np.array_equal(Yh, Wx[ks])
    Wh = oracle.dequantize(qw, sc, ze, mode=mode).view(np.float16).astype(np.float64)
    assert np.array_equal(Wx.astype(np.float16).astype(np.float64), Wh)     # one rounding of the exact weight
    Xd = X.view(np.float16).astype(np.float64)
    Ye = oracle.gemm_exact(X, qw, sc, ze, mode=mode, nthreads=3)
    assert np.allclose(Ye, Xd @ Wx, rtol=1e-12, atol=1e-12)
    Y16 = oracle.gemm(X, qw, sc, ze, mode=mode)
    ulp = np.spacing(np.abs(Wh).astype(np.float16)).astype(np.float64)      # fp16 ulp of each w_hat
    bound = np.abs(Xd) @ (ulp / 2)
    assert np.all(np.abs(Ye - Y16) <= bound * (1 + 1e-9) + 1e-12)
    assert np.any(Ye != Y16)                                                 # the definitions do differ


def test_gemm_transposition_sensitive():
    # a transposed operand (using W_hat[n][k]) or swapped X rows would change this product
    K, N = 256, 256
    W = synth.host(2, 2, synth.WEIGHT, K, N)
    X = synth.host(2, 4, synth.ACT, 3, K)
    qw, sc, ze, st = oracle.quantize(W)
    Wh = oracle.dequantize(qw, sc, ze).view(np.float16).astype(np.float64)
    Y = oracle.gemm(X, qw, sc, ze)
    Xd = X.view(np.float16).astype(np.float64)
    assert not np.allclose(Y, Xd @ Wh.T)
    assert np.allclose(Y, Xd @ Wh)


# ---------------------------------------------------------------------------------------------------
# Acceptance — golden worked example, SPEC examples, brute force, losslessness vs AR decoding.
# ---------------------------------------------------------------------------------------------------
def test_accept_golden_8node():
    g = _read_golden("accept_8node.txt")
    t = [int(x) for x in g["tokens"][0]]
    p = [int(x) for x in g["parents"][0]]
    a = [int(x) for x in g["argmax"][0]]
    L, bonus, st, path, _ = oracle.accept(t, p, a)
    assert (L, bonus, st) == (int(g["len"][0][0]), int(g["bonus"][0][0]), oracle.DEV_OK)
    assert path == [int(x) for x in g["path"][0]]


def test_accept_spec_sequence_examples():
    d = 6
    cont = [5, 9, 2, 7, 7, 1, 3]                       # target's greedy continuation after the root
    toks = [42] + cont[:d]
    par = [-1] + list(range(d))
    argmax = cont[:d + 1]                               # argmax at node i = next greedy token
    assert oracle.accept(toks, par, argmax)[:3] == (d, cont[d], 0)      # S:292 perfect draft: all d accepted
    bad = list(toks)
    bad[1] = 99
    assert oracle.accept(bad, par, argmax)[:3] == (0, cont[0], 0)       # S:293 draft[0] wrong: 0 + bonus


def test_accept_spec_tree_examples():
    # S:301 single-chain tree matching the greedy continuation -> whole chain accepted
    assert oracle.accept([0, 4, 5, 6], [-1, 0, 1, 2], [4, 5, 6, 8])[:3] == (3, 8, 0)
    # S:302 no child of the root matches the target argmax -> 0 accepted, bonus = argmax at root
    assert oracle.accept([0, 4, 5, 6], [-1, 0, 0, 0], [9, 1, 1, 1])[:3] == (0, 9, 0)


def test_accept_m1_equals_autoregressive_step():
    # verification width 1 (root only) is exactly one AR decode step: nothing accepted, bonus = argmax
    for a in [0, 17, 128255]:
        assert oracle.accept([3], [-1], [a])[:4] == (0, a, 0, [])


def test_accept_bad_trees():
    for p in ([0, 0], [-1, 1], [-1, 0, 3], [-1, -1]):
        L, bonus, st, path, out = oracle.accept([1] * len(p), p, [1] * len(p))
        assert (L, bonus, st) == (0, -1, oracle.DEV_BAD_TREE) and np.all(out[3:] == -1)


def _all_trees(n):
    """All parent vectors with parents[i] < i for n nodes."""
    for ps in itertools.product(*[range(i) for i in range(1, n)]):
        yield [-1] + list(ps)


def test_accept_brute_force_small_trees():
    # enumerate every root->node path; valid iff each edge matches; choose longest, ties smallest end node
    rng = np.random.default_rng(7)
    count = 0
    for n in range(1, 8):
        for par in _all_trees(n):
            for _ in range(3):
                tok = rng.integers(0, 3, n).tolist()
                am = rng.integers(0, 3, n).tolist()
                best = (0, 0)
                for end in range(n):
                    path, x = [], end
                    while x != 0:
                        path.append(x)
                        x = par[x]
                    path.reverse()
                    prev, ok = 0, True
                    for c in path:
                        ok &= tok[c] == am[prev]
                        prev = c
                    if ok and len(path) > best[0]:
                        best = (len(path), end)
                L, bonus, st, got_path, _ = oracle.accept(tok, par, am)
                assert (L, bonus) == (best[0], am[best[1]])
                count += 1
    assert count > 1000


def test_accept_lossless_vs_autoregressive_decoding():
    # A deterministic "target" f(context) -> next token. Build random trees whose node tokens are sometimes the
    # target's greedy token; argmax[i] = f(context of i). The accepted tokens + bonus must equal the first
    # len+1 tokens of AR greedy decoding, and no tree path may match a longer AR prefix (losslessness).
    rng = np.random.default_rng(99)

    def f(ctx):
        h = 1469598103934665603
        for t in ctx:
            h = ((h ^ t) * 1099511628211) & 0xFFFFFFFFFFFF
        return h % 5

    for trial in range(400):
        n = int(rng.integers(1, 40))
        par = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
        prefix = [int(x) for x in rng.integers(0, 5, 3)]
        toks, ctx = [prefix[-1]], [prefix]
        for i in range(1, n):
            c = ctx[par[i]]
            t = f(c) if rng.random() < 0.6 else int(rng.integers(0, 5))
            toks.append(t)
            ctx.append(c + [t])
        am = [f(c) for c in ctx]
        L, bonus, st, path, _ = oracle.accept(toks, par, am)
        # AR rollout from the prefix
        ar, c = [], list(prefix)
        for _ in range(n + 1):
            t = f(c)
            ar.append(t)
            c.append(t)
        assert [toks[i] for i in path] + [bonus] == ar[:L + 1]
        # maximality: no node's context extends the AR prefix beyond L
        for i in range(n):
            d = len(ctx[i]) - len(prefix)
            if ctx[i][len(prefix):] == ar[:d]:
                assert d <= L


# ---------------------------------------------------------------------------------------------------
# LM head + greedy argmax: pins against numpy, closed forms, ties, planted winners
# ---------------------------------------------------------------------------------------------------
def test_lmhead_argmax_matches_numpy_float64():
    # library routine: float64 matmul of the same fp16 values, argmax (first maximum); K != V catches a
    # transposed operand
    rng = np.random.default_rng(11)
    for M, K, V in ((1, 128, 77), (5, 384, 1000), (13, 256, 333)):
        H = rng.standard_normal((M, K)).astype(np.float16)
        W = (0.05 * rng.standard_normal((V, K))).astype(np.float16)
        idx, val, lg = oracle.lmhead_argmax(H, W, nthreads=3, want_logits=True)
        ref = H.astype(np.float64) @ W.astype(np.float64).T
        assert np.allclose(lg, ref, rtol=0, atol=1e-9)
        assert np.array_equal(idx, np.argmax(ref, axis=1))
        assert np.allclose(val, ref.max(axis=1), rtol=0, atol=1e-9)


def test_lmhead_argmax_closed_form_and_ties():
    K, V = 256, 64
    H = np.ones((2, K), dtype=np.float16)
    c = np.array([(v * 37) % 64 - 20 for v in range(V)], dtype=np.float64) / 64.0   # exact fp16 values
    W = np.repeat(c[:, None], K, axis=1).astype(np.float16)
    idx, val = oracle.lmhead_argmax(H, W)
    assert np.all(val == K * c.max())                       # logit = K * c_v exactly
    assert np.all(idx == int(np.argmax(c)))
    # exact ties -> lowest id: duplicate the winning row at a lower and a higher id
    W2 = W.copy()
    w = int(np.argmax(c))
    W2[w + 5] = W2[w]
    W2[3] = W2[w]
    idx2, _ = oracle.lmhead_argmax(H, W2)
    assert np.all(idx2 == min(3, w))
    # all-zero head: every logit 0, the lowest id wins
    idx3, val3 = oracle.lmhead_argmax(H, np.zeros((V, K), dtype=np.float16))
    assert np.all(idx3 == 0) and np.all(val3 == 0)


def test_lmhead_argmax_planted_winner_and_thread_invariance():
    rng = np.random.default_rng(12)
    M, K, V = 6, 512, 900
    H = rng.standard_normal((M, K)).astype(np.float16)
    W = (0.02 * rng.standard_normal((V, K))).astype(np.float16)
    plant = rng.choice(V, size=M, replace=False)
    for m, v in enumerate(plant):
        W[v] = (H[m].astype(np.float32) * 0.5).astype(np.float16)    # logit ~ 0.5 |h|^2 >> the rest
    idx1, val1 = oracle.lmhead_argmax(H, W, nthreads=1)
    idx7, val7 = oracle.lmhead_argmax(H, W, nthreads=7)
    assert np.array_equal(idx1, plant)
    assert np.array_equal(idx1, idx7) and np.array_equal(val1, val7)


# ---------------------------------------------------------------------------------------------------
# Tree-masked verify attention + KV compaction
# ---------------------------------------------------------------------------------------------------
def _attn_inputs(rng, M, L, Hq, Hkv, D, scale=1.0):
    Q = (scale * rng.standard_normal((M, Hq, D))).astype(np.float16)
    K = (scale * rng.standard_normal((L + M, Hkv, D))).astype(np.float16)
    V = rng.standard_normal((L + M, Hkv, D)).astype(np.float16)
    return Q, K, V


def _dense_masked_attention(Q, K, V, mask):
    # numpy float64: explicit boolean mask [M, L+M], softmax over the visible rows (library-routine formulation)
    M, Hq, D = Q.shape
    Hkv = K.shape[1]
    g = Hq // Hkv
    Qf, Kf, Vf = Q.astype(np.float64), K.astype(np.float64), V.astype(np.float64)
    O = np.zeros((M, Hq, D))
    for h in range(Hq):
        S = Qf[:, h, :] @ Kf[:, h // g, :].T / np.sqrt(D)
        S = np.where(mask, S, -np.inf)
        P = np.exp(S - S.max(axis=1, keepdims=True))
        P /= P.sum(axis=1, keepdims=True)
        O[:, h, :] = P @ Vf[:, h // g, :]
    return O


def test_tree_attention_sequence_draft_is_causal_attention():
    rng = np.random.default_rng(21)
    M, L, Hq, Hkv, D = 7, 40, 8, 2, 64
    Q, K, V = _attn_inputs(rng, M, L, Hq, Hkv, D)
    mask = np.zeros((M, L + M), dtype=bool)
    mask[:, :L] = True
    mask[:, L:] = np.tril(np.ones((M, M), dtype=bool))      # causal over the new rows
    O = oracle.tree_attention(Q, K, V, np.arange(-1, M - 1))
    assert np.allclose(O, _dense_masked_attention(Q, K, V, mask), rtol=0, atol=1e-12)


def test_tree_attention_equals_its_root_to_node_path_as_a_sequence():
    # path invariance: node i of a tree sees exactly what the last row of the sequence (root .. i) sees
    rng = np.random.default_rng(22)
    M, L, Hq, Hkv, D = 12, 17, 4, 2, 32
    Q, K, V = _attn_inputs(rng, M, L, Hq, Hkv, D)
    par = [-1, 0, 0, 1, 1, 2, 3, 3, 5, 8, 0, 10]
    O = oracle.tree_attention(Q, K, V, par)
    for i in range(M):
        path = []
        a = i
        while a != -1:
            path.append(a)
            a = par[a]
        path = path[::-1]
        n = len(path)
        Qs = Q[path]
        Ks = np.concatenate([K[:L], K[[L + p for p in path]]])
        Vs = np.concatenate([V[:L], V[[L + p for p in path]]])
        Os = oracle.tree_attention(Qs, Ks, Vs, np.arange(-1, n - 1))
        assert np.allclose(O[i], Os[-1], rtol=0, atol=1e-12)


def test_tree_attention_closed_forms_and_gqa_mapping():
    rng = np.random.default_rng(23)
    M, L, Hq, Hkv, D = 5, 0, 4, 2, 16
    Q, K, V = _attn_inputs(rng, M, L, Hq, Hkv, D)
    par = [-1, 0, 1, 1, 0]
    O = oracle.tree_attention(Q, K, V, par)
    assert np.array_equal(O[0], V[0][[h // 2 for h in range(Hq)]].astype(np.float64))   # root, empty prefix
    # equal keys -> uniform weights -> mean of the visible values (node 3 sees rows 0, 1, 3)
    K2 = np.repeat(K[:1], L + M, axis=0)
    O2 = oracle.tree_attention(Q, K2, V, par)
    vis = [0, 1, 3]
    assert np.allclose(O2[3], V[vis].astype(np.float64).mean(axis=0)[[h // 2 for h in range(Hq)]], rtol=0, atol=1e-12)
    # heads of one group share the kv head; identical queries in different groups differ
    Q3 = Q.copy()
    Q3[:, 1] = Q3[:, 0]
    Q3[:, 2] = Q3[:, 0]
    O3 = oracle.tree_attention(Q3, K, V, par)
    assert np.array_equal(O3[:, 0], O3[:, 1])
    assert not np.allclose(O3[:, 0], O3[:, 2])


def test_kv_compact_worked_example_and_chain_equivalence():
    rng = np.random.default_rng(24)
    L, Hq, Hkv, D = 9, 4, 2, 16
    tok = [100, 11, 12, 21, 22, 23, 31, 32]
    par = [-1, 0, 0, 1, 1, 2, 3, 5]
    am = [12, 99, 23, 31, 99, 32, 99, 40]
    acc = oracle.accept(tok, par, am)[4]            # accepted path [2, 5, 7] (tests/golden/accept_8node.txt)
    assert list(acc[3:6]) == [2, 5, 7] and acc[0] == 3
    M = len(tok)
    Q, K, V = _attn_inputs(rng, M + 1, L, Hq, Hkv, D)
    K, V = K[:L + M], V[:L + M]
    Kc, Vc = oracle.kv_compact(K, V, L, acc)
    assert np.array_equal(Kc[:L + 1], K[:L + 1]) and np.array_equal(Vc[:L + 1], V[:L + 1])
    for k, p in enumerate([2, 5, 7], start=1):
        assert np.array_equal(Kc[L + k], K[L + p]) and np.array_equal(Vc[L + k], V[L + p])
    # the next token (bonus position) attends prefix + root + path: on the compacted cache it is a sequence
    # row; on the original tree it is a new child of the accepted leaf (node 7)
    qn, kn, vn = Q[M:M + 1], rng.standard_normal((1, Hkv, D)).astype(np.float16), rng.standard_normal((1, Hkv, D)).astype(np.float16)
    n = 1 + 3
    Kseq = np.concatenate([Kc[:L + n], kn])
    Vseq = np.concatenate([Vc[:L + n], vn])
    Oseq = oracle.tree_attention(np.concatenate([Q[[0, 2, 5, 7]], qn]), Kseq, Vseq, np.arange(-1, n))
    Otree = oracle.tree_attention(np.concatenate([Q[:M], qn]), np.concatenate([K, kn]), np.concatenate([V, vn]), par + [7])
    assert np.allclose(Oseq[-1], Otree[-1], rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------------------------------
# Block Hadamard rotation of W4A16+Rot
# ---------------------------------------------------------------------------------------------------
def test_hadamard_matches_scipy_and_is_orthogonal():
    import scipy.linalg
    rng = np.random.default_rng(31)
    for B, K in ((8, 32), (64, 128), (128, 512)):
        X = rng.standard_normal((3, K)).astype(np.float16)
        Y = oracle.hadamard(X, B)
        H = scipy.linalg.hadamard(B).astype(np.float64) / np.sqrt(B)      # library routine (Sylvester order)
        ref = np.concatenate([X[:, b:b + B].astype(np.float64) @ H.T for b in range(0, K, B)], axis=1)
        assert np.allclose(Y, ref, rtol=0, atol=1e-12)
        # orthogonal and symmetric: applying it twice gives the input back (to fp64 rounding)
        Y2 = np.concatenate([Y[:, b:b + B] @ H.T for b in range(0, K, B)], axis=1)
        assert np.allclose(Y2, X.astype(np.float64), rtol=0, atol=1e-12)
    # a basis vector maps to a scaled Hadamard column
    e = np.zeros((1, 128), dtype=np.float16)
    e[0, 5] = 1
    assert np.allclose(oracle.hadamard(e, 128)[0], scipy.linalg.hadamard(128)[:, 5] / np.sqrt(128), rtol=0, atol=0)


def test_hadamard_rotation_leaves_the_product_invariant():
    # x W = (x H)(H^T W): the rotation is folded into the weights offline, applied to activations online
    import scipy.linalg
    rng = np.random.default_rng(32)
    K, N, B = 256, 40, 128
    X = rng.standard_normal((4, K)).astype(np.float16)
    W = rng.standard_normal((K, N))
    H = scipy.linalg.hadamard(B) / np.sqrt(B)
    HW = np.concatenate([H @ W[b:b + B] for b in range(0, K, B)], axis=0)   # H symmetric: H^T = H
    assert np.allclose(oracle.hadamard(X, B) @ HW, X.astype(np.float64) @ W, rtol=0, atol=1e-10)
