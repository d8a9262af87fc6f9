"""CPU side of the in-chain tensor-parallel all-reduce (include/w4a16.h W4A16_OP_ALLREDUCE):
the oracle's sum pinned to independent facts, and w4a16_chain_plan's validation of ALLREDUCE ops (group,
region bounds, the cyclic read-before-rewrite rule) — planning an ALLREDUCE / SILU_MUL-only chain touches no
device, so it runs here with placeholder addresses that are never dereferenced."""
import ctypes

import numpy as np
import pytest

import oracle


# ---------------- oracle pins ----------------

def test_allreduce_oracle_exact_on_integers_and_identity():
    rng = np.random.default_rng(0)
    for T in (1, 2, 4, 8):
        P = rng.integers(-200, 200, size=(T, 1000)).astype(np.float16)   # integers: every sum is exact in fp16
        got = oracle.allreduce(P).view(np.float16).astype(np.float64)
        assert np.array_equal(got, P.astype(np.float64).sum(axis=0))
    P = rng.standard_normal((1, 500)).astype(np.float16)
    assert np.array_equal(oracle.allreduce(P), P[0].view(np.uint16))                 # T = 1: identity
    Q = np.stack([P[0], -P[0]])
    assert not np.any(oracle.allreduce(Q).view(np.float16).astype(np.float64))      # x + (-x) = 0


def test_allreduce_oracle_matches_numpy_fp64_sum_rounded_once():
    rng = np.random.default_rng(1)
    for T in (2, 3, 8):
        P = (rng.standard_normal((T, 4096)) * rng.choice([1e-3, 1, 300], size=(T, 1))).astype(np.float16)
        ref = P.astype(np.float64).sum(axis=0).astype(np.float16)   # numpy's own fp64 -> fp16 RNE conversion
        assert np.array_equal(oracle.allreduce(P), ref.view(np.uint16))
    # order matters for a single-rounded sum only through rounding: the oracle is order-free (exact fp64)
    P = np.array([[2048.0], [1.0], [1.0]], dtype=np.float16)   # 2048 + 1 + 1: fp16 left-to-right gives 2048
    assert oracle.allreduce(P).view(np.float16)[0] == np.float16(2050.0)


# ---------------- plan validation (no device) ----------------

def _w4():
    try:
        import paper_2505_22179_b200 as w4
        from paper_2505_22179_b200 import _lib
    except ImportError as e:   # pragma: no cover - the library is built by `make`
        pytest.skip(f"libw4a16.so not built: {e}")
    return w4, _lib


BASE = 0x7f0000000000   # placeholder region addresses (never dereferenced by the planner)
REGION = 1 << 20


def _group(world=2, rank=0, slots=4, bases=None):
    w4, L = _w4()
    g = L.W4A16PeerGroup()
    for q in range(world):
        g.base[q] = (bases or [BASE + q * (1 << 24) for q in range(world)])[q]
    g.bytes, g.flag_offset, g.flag_slots, g.world, g.rank = REGION, 0, slots, world, rank
    return g


def _plan(ops, M=8, sms=148):
    # the planner's validation (w4a16_chain_plan's rules) without tensor-map encoding, which needs a GPU
    w4, L = _w4()
    arr = (L.W4A16Op * len(ops))(*ops)
    return L.lib.w4a16_chain_check_sms(ctypes.addressof(arr), len(ops), M, -1, sms)


def _ar(g, x_off, y, N=1024, rank=0):
    _, L = _w4()
    return L.W4A16Op(L.W4A16_OP_ALLREDUCE, g.base[rank] + x_off, ctypes.addressof(g), y, N, N, 0)


def _silu(gu, out, N=1024):
    _, L = _w4()
    return L.W4A16Op(L.W4A16_OP_SILU_MUL, gu, None, out, 2 * N, N, 0)


PACKED = 0x7d0000000000   # placeholder weight blob (never dereferenced by the planner)


def _gemm(x, y, N=1024, K=4096):
    # the row-parallel GEMM whose Y is the ALLREDUCE's partial (the op right before it)
    _, L = _w4()
    return L.W4A16Op(L.W4A16_OP_GEMM, x, PACKED, y, K, N, 0)


OUT = 0x7e0000000000   # ordinary (non-region) buffers
P1, P2 = 65536, 131072  # partial buffers inside the region, after the flag area


def test_flag_area_size():
    w4, L = _w4()
    assert L.lib.w4a16_peer_flag_bytes(0) == 0
    for slots in (1, 4, 160):
        nb = L.lib.w4a16_peer_flag_bytes(slots)
        assert nb % 256 == 0 and nb >= (16 + slots * L.W4A16_AR_MAX_TILES) * 4


def test_plan_accepts_alternating_partials():
    g = _group()
    # layer: producer -> P1, AR(P1 -> out1), producer -> P2, AR(P2 -> out2), repeated (cyclic rule holds)
    ops = [_gemm(OUT, g.base[0] + P1), _ar(g, P1, OUT + (1 << 20)),
           _gemm(OUT + (2 << 20), g.base[0] + P2), _ar(g, P2, OUT + (3 << 20))]
    assert _plan(ops) == 0


def test_plan_multicast_group_needs_no_peer_mappings():
    g = _group()
    g.base[1] = None                     # the NVLS path never maps the peers' regions
    ops = [_gemm(OUT, g.base[0] + P1), _ar(g, P1, OUT + (1 << 20)),
           _gemm(OUT + (2 << 20), g.base[0] + P2), _ar(g, P2, OUT + (3 << 20))]
    assert _plan(ops) != 0               # peer-load path: every mapping is needed
    g.mc_base = BASE + (1 << 30)
    assert _plan(ops) == 0


def test_plan_rejects_allreduce_not_fused_with_its_gemm():
    g = _group()
    # the op before an ALLREDUCE must be the GEMM that writes exactly its partial
    ops = [_silu(OUT, g.base[0] + P1), _ar(g, P1, OUT + (1 << 20)),
           _gemm(OUT + (2 << 20), g.base[0] + P2), _ar(g, P2, OUT + (3 << 20))]
    assert _plan(ops) != 0
    ops = [_gemm(OUT, g.base[0] + P1 + 256), _ar(g, P1, OUT + (1 << 20)),
           _gemm(OUT + (2 << 20), g.base[0] + P2), _ar(g, P2, OUT + (3 << 20))]
    assert _plan(ops) != 0


def test_plan_rejects_rewrite_before_another_allreduce():
    g = _group()
    # one partial buffer, one AR per run: the next run's producer rewrites P1 while peers may still read it
    ops = [_gemm(OUT, g.base[0] + P1), _ar(g, P1, OUT + (1 << 20))]
    assert _plan(ops) != 0
    # rewritten inside the same run right after its AR
    ops = [_gemm(OUT, g.base[0] + P1), _ar(g, P1, OUT + (1 << 20)), _gemm(OUT + (2 << 20), g.base[0] + P1),
           _ar(g, P1, OUT + (3 << 20))]
    assert _plan(ops) != 0


@pytest.mark.parametrize("case", ["outside", "flags", "world", "rank", "slots", "two_groups", "shape"])
def test_plan_rejects_bad_allreduce(case):
    g = _group()
    good = lambda gg=g: [_gemm(OUT, gg.base[0] + P1), _ar(gg, P1, OUT + (1 << 20)),
                         _gemm(OUT + (2 << 20), gg.base[0] + P2), _ar(gg, P2, OUT + (3 << 20))]
    ops = good()
    if case == "outside":
        ops[0] = _gemm(OUT, g.base[0] + REGION - 1024)
        ops[1] = _ar(g, REGION - 1024, OUT + (1 << 20))          # P runs past the region end
    elif case == "flags":
        ops[0] = _gemm(OUT, g.base[0])
        ops[1] = _ar(g, 0, OUT + (1 << 20))                      # P overlaps the flag area
    elif case == "world":
        g.world = 9
    elif case == "rank":
        g.rank = 2
    elif case == "slots":
        g.flag_slots = 1                                          # two AR ops, one slot
    elif case == "two_groups":
        g2 = _group()
        ops[3] = _ar(g2, P2, OUT + (3 << 20))
    elif case == "shape":
        ops[1].K = 512                                            # K must equal N
    assert _plan(ops) != 0
