"""Chains (include/w4a16.h w4a16_chain_plan / w4a16_chain_run): a sequence of GEMM and SiLU*mul ops in one
persistent launch must give exactly what the same ops launched one by one give (same family, same split
plan, same reduction order: bit-identical), honour RAW / WAR / WAW dependencies through shared buffers,
re-arm its counters for the next run, and be CUDA-graph capturable. The single-op kernels are themselves
checked against the oracle (tests/test_gpu_parity.py); one chain op is re-checked against it here too."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _w4():
    import paper_2505_22179_b200 as w4
    return w4


def _u16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _mlp(H=2048, F=2560, layers=2, seed=0, mode=0):
    w4 = _w4()
    mats = []
    for l in range(layers):
        gu = w4.pack_linear(synth.gpu(seed, 1000 + 2 * l, synth.WEIGHT, H, 2 * F), mode=mode)
        dn = w4.pack_linear(synth.gpu(seed, 1001 + 2 * l, synth.WEIGHT, F, H), mode=mode)
        mats.append((gu, dn))
    return mats


def _mlp_ops(mats, x, gu_buf, act, y):
    # layer l: GU = x_l . W_gu ; act = silu(gate) * up ; y = act . W_down ; x_{l+1} = y  (RAW through y,
    # WAR on GU / act across layers, WAW on y)
    ops = []
    cur = x
    for gu, dn in mats:
        ops += [("gemm", cur, gu, gu_buf), ("silu_mul", gu_buf, act), ("gemm", act, dn, y)]
        cur = y
    return ops


def _run_eager(ops, family, ws):
    w4 = _w4()
    for op in ops:
        if op[0] == "gemm":
            _, X, pl, Y = op
            pl(X, Y, ws, family=family)
        else:
            _, GU, out = op
            w4.w4a16_silu_mul(GU, out)
    torch.cuda.synchronize()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("M,family", [(M, f) for f in (0, 2) for M in (1, 5, 8, 9, 16)])
def test_chain_mlp_stack_bit_exact_vs_single_ops(M, family):
    w4 = _w4()
    H, F = 2048, 2560
    mats = _mlp(H, F, layers=3, seed=M)
    f16 = dict(dtype=torch.float16, device="cuda")
    x = synth.gpu(7, 5, synth.ACT, M, H)
    bufs_e = [torch.full((M, 2 * F), float("nan"), **f16), torch.full((M, F), float("nan"), **f16), torch.empty((M, H), **f16)]
    bufs_c = [torch.full((M, 2 * F), float("nan"), **f16), torch.full((M, F), float("nan"), **f16), torch.empty((M, H), **f16)]
    # eager reference: every op launched on its own (x must not be overwritten: first layer reads x only)
    ws = w4.alloc_workspace(M, [(H, 2 * F), (F, H)])
    x_e, x_c = x.clone(), x.clone()
    _run_eager(_mlp_ops(mats, x_e, *bufs_e), family, ws)
    ch = w4.Chain(_mlp_ops(mats, x_c, *bufs_c), M, family=family)
    for rep in range(3):   # counters re-armed after every run
        bufs_c[2].zero_()
        ch()
        torch.cuda.synchronize()
        for a, b in zip(bufs_e, bufs_c):
            assert np.array_equal(_u16(a), _u16(b)), f"rep {rep}"


@pytest.mark.timeout(300)
def test_chain_independent_gemms_match_single_and_oracle():
    # several shapes, no dependencies, the last op re-checked against the fp64 oracle
    w4 = _w4()
    M = 7
    shapes = [(4096, 2560), (2048, 8192), (8192, 1024), (5120, 4096)]
    ops, ref_ys, mats = [], [], []
    ws = w4.alloc_workspace(M, shapes)
    for i, (K, N) in enumerate(shapes):
        W = synth.host(3, 200 + i, synth.WEIGHT, K, N)
        pl = w4.pack_linear(torch.from_numpy(W.view(np.int16)).cuda().view(torch.float16))
        X = synth.gpu(3, 300 + i, synth.ACT, M, K)
        Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
        Ye = torch.empty_like(Y)
        pl(X, Ye, ws, family=0)
        ops.append(("gemm", X, pl, Y))
        ref_ys.append(Ye)
        mats.append((W, X))
    ch = w4.Chain(ops, M, family=0)
    ch()
    torch.cuda.synchronize()
    for (_, _, _, Y), Ye in zip(ops, ref_ys):
        assert np.array_equal(_u16(Y), _u16(Ye))
    W, X = mats[-1]
    qw, sc, ze, _ = oracle.quantize(W)
    ref = oracle.gemm(_u16(X), qw, sc, ze)
    y = ops[-1][3].float().cpu().numpy().astype(np.float64)
    assert np.all(np.abs(y - ref) <= 1e-2 * (1 + np.abs(ref)))


@pytest.mark.timeout(300)
def test_chain_graph_capture_and_replay():
    w4 = _w4()
    M, H, F = 16, 2048, 2560
    mats = _mlp(H, F, layers=2, seed=4)
    f16 = dict(dtype=torch.float16, device="cuda")
    x = synth.gpu(9, 5, synth.ACT, M, H)
    bufs = [torch.empty((M, 2 * F), **f16), torch.empty((M, F), **f16), torch.empty((M, H), **f16)]
    ch = w4.Chain(_mlp_ops(mats, x, *bufs), M)
    ch()
    torch.cuda.synchronize()
    want = _u16(bufs[2])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ch(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ch(s)
    bufs[2].zero_()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(_u16(bufs[2]), want)


def test_chain_rejects_bad_ops():
    w4 = _w4()
    M = 8
    pl = w4.pack_linear(synth.gpu(0, 1, synth.WEIGHT, 2048, 2560))
    X = torch.zeros((M, 2048), dtype=torch.float16, device="cuda")
    Y = torch.zeros((M, 2560), dtype=torch.float16, device="cuda")
    with pytest.raises(w4.W4A16Error):
        w4.Chain([("gemm", X, pl, Y)], 17)           # chains serve M <= 16 (the mma.sync families)
    small = w4.pack_linear(synth.gpu(0, 2, synth.WEIGHT, 256, 256))
    with pytest.raises(w4.W4A16Error):               # fewer units than CTAs
        w4.Chain([("gemm", X[:, :256].contiguous(), small, Y[:, :256].contiguous())], M)
    buf = torch.zeros(M * 4096, dtype=torch.float16, device="cuda")
    sq = w4.pack_linear(synth.gpu(0, 3, synth.WEIGHT, 2048, 2048))
    with pytest.raises(w4.W4A16Error):               # in place (X and Y overlap)
        w4.Chain([("gemm", buf[:M * 2048].view(M, 2048), sq, buf[M * 1024:M * 3072].view(M, 2048))], M)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("M,family", [(1, 0), (8, 0), (13, 2), (16, 0)])
def test_chain_fused_silu_matches_gemm_then_blocked_silu(M, family):
    # W4A16_OP_GEMM_SILU (gate-up weight in [64 gate | 64 up] tiles, SiLU*mul in the GEMM epilogue) against
    # the same gate-up GEMM launched alone followed by w4a16_silu_mul_blocked(block = 64): bit-identical, also
    # across layers (the down GEMM reads the fused output tile by tile), and act itself against numpy on the
    # host-side unfused values
    w4 = _w4()
    H, F = 2048, 2560
    mats = _mlp(H, F, layers=2, seed=M + 11)
    f16 = dict(dtype=torch.float16, device="cuda")
    x = synth.gpu(8, 5, synth.ACT, M, H)
    ws = w4.alloc_workspace(M, [(H, 2 * F), (F, H)])
    gu_e, act_e, y_e = torch.empty((M, 2 * F), **f16), torch.empty((M, F), **f16), torch.empty((M, H), **f16)
    cur = x
    for gu, dn in mats:
        gu(cur, gu_e, ws, family=family)
        w4.w4a16_silu_mul_blocked(gu_e, act_e, 64)
        dn(act_e, y_e, ws, family=family)
        cur = y_e.clone()
    torch.cuda.synchronize()
    # blocked SiLU*mul against an fp32 reference of its definition (include/w4a16.h)
    g = gu_e.float().view(M, F // 64, 2, 64)
    ref = (g[:, :, 0] / (1 + torch.exp(-g[:, :, 0])) * g[:, :, 1]).reshape(M, F)
    assert torch.allclose(act_e.float(), ref, rtol=2e-3, atol=1e-3)
    act_c, y_c, y_mid = torch.empty((M, F), **f16), torch.empty((M, H), **f16), torch.empty((M, H), **f16)
    (gu0, dn0), (gu1, dn1) = mats
    ops = [("gemm_silu", x, gu0, act_c), ("gemm", act_c, dn0, y_mid), ("gemm_silu", y_mid, gu1, act_c),
           ("gemm", act_c, dn1, y_c)]
    ch = w4.Chain(ops, M, family=family)
    for rep in range(2):
        ch()
        torch.cuda.synchronize()
        assert np.array_equal(_u16(act_c), _u16(act_e)), rep
        assert np.array_equal(_u16(y_c), _u16(y_e)), rep


@pytest.mark.timeout(300)
def test_chains_of_different_M_share_one_workspace():
    # chains at M <= 8 and M = 9..16 lay their op counts out with different strides but keep the run number and
    # exit counter at fixed offsets (gemm_mma.cu kDSMax), so chains of any M may share one workspace: run them
    # alternately on one workspace and compare each run with the op-by-op launches, bit for bit
    w4 = _w4()
    H, F = 2048, 2560
    mats = _mlp(H, F, layers=2, seed=77)
    f16 = dict(dtype=torch.float16, device="cuda")
    cases = {}
    for M in (8, 16):
        x = synth.gpu(7, 50 + M, synth.ACT, M, H)
        bufs_e = [torch.empty((M, 2 * F), **f16), torch.empty((M, F), **f16), torch.empty((M, H), **f16)]
        bufs_c = [torch.empty((M, 2 * F), **f16), torch.empty((M, F), **f16), torch.empty((M, H), **f16)]
        ws = w4.alloc_workspace(M, [(H, 2 * F), (F, H)])
        _run_eager(_mlp_ops(mats, x.clone(), *bufs_e), 0, ws)
        cases[M] = (x.clone(), bufs_e, bufs_c)
    shared = None
    chains = {}
    for M in (8, 16):
        x_c, _, bufs_c = cases[M]
        probe = w4.Chain(_mlp_ops(mats, x_c, *bufs_c), M)
        if shared is None or probe.ws.numel() > shared.numel():
            shared = torch.zeros(max(probe.ws.numel(), 0 if shared is None else shared.numel()), dtype=torch.uint8, device="cuda")
    for M in (8, 16):
        x_c, _, bufs_c = cases[M]
        chains[M] = w4.Chain(_mlp_ops(mats, x_c, *bufs_c), M, workspace=shared)
    for rep in range(3):
        for M in (8, 16, 16, 8):
            _, bufs_e, bufs_c = cases[M]
            for b in bufs_c:
                b.fill_(float("nan"))
            chains[M]()
            torch.cuda.synchronize()
            for a, b in zip(bufs_e, bufs_c):
                assert np.array_equal(_u16(a), _u16(b)), (rep, M)
