"""In-chain tensor-parallel all-reduce (include/w4a16.h W4A16_OP_ALLREDUCE).

The round's GPU box has one GPU, so t-way tensor parallelism is simulated on it: T chains, one per
simulated rank, each planned for SMs/T SMs and launched side by side on T streams (non-cooperatively; the
grids together fit the device), with T symmetric regions on the same device as the "peers". The kernel
code is the multi-GPU code: flags through st.release.sys / ld.acquire.sys, partials read through the peer
pointers. Two row-parallel layers per run (GEMM -> ALLREDUCE -> GEMM on the reduced output -> ALLREDUCE)
exercise the ready flags, the run counter across repeated runs, RAW dependencies on an ALLREDUCE output,
and the alternating-partials rule. Checked: every rank's output identical; each output equal to its
defined arithmetic (fp32 sum in rank order of the fp16 partials, rounded once) bit for bit; within one
fp16 ulp of the oracle's fp64 sum; each partial within the GEMM tolerance of the oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _u16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _fp32_rank_sum(parts):
    acc = np.zeros(parts[0].shape, dtype=np.float32)
    for p in parts:                      # rank order, fp32, one rounding at the end (header definition)
        acc = acc + p.float().cpu().numpy()
    return acc.astype(np.float16).view(np.uint16)


def _oracle_gemm(X, W, mode):
    qw, sc, ze, _ = oracle.quantize(W, mode=mode)
    return oracle.gemm(_u16(X), qw, sc, ze, mode=mode)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("T,M,mode", [(1, 8, 0), (2, 8, 0), (2, 1, 0), (2, 13, 1), (4, 16, 0), (4, 5, 0)])
def test_chain_allreduce_simulated_ranks(T, M, mode):
    import paper_2505_22179_b200 as w4
    sms = torch.cuda.get_device_properties(0).multi_processor_count // T
    # rank-local K shard of layer 1; layer 2 reads the reduced [M, H]; every CTA owns >= 1 unit of every GEMM
    H = 1280
    Kr = H2 = max(1024, 128 * -(-sms // (H // 128)))
    f16 = dict(dtype=torch.float16, device="cuda")
    groups = w4.PeerGroup.simulated(T, 1 << 20, flag_slots=4, device="cuda")
    Wa = [synth.host(11, 100 + r, synth.WEIGHT, Kr, H) for r in range(T)]
    Wb = [synth.host(11, 200 + r, synth.WEIGHT, H, H2) for r in range(T)]
    ranks = []
    for r, g in enumerate(groups):
        pa = w4.pack_linear(torch.from_numpy(Wa[r].view(np.int16)).cuda().view(torch.float16), mode=mode)
        pb = w4.pack_linear(torch.from_numpy(Wb[r].view(np.int16)).cuda().view(torch.float16), mode=mode)
        X = torch.empty((M, Kr), **f16)
        P1, P2 = g.alloc(M, H), g.alloc(M, H2)
        Y1, Y2 = torch.empty((M, H), **f16), torch.empty((M, H2), **f16)
        ops = [("gemm", X, pa, P1), ("allreduce", P1, Y1, g), ("gemm", Y1, pb, P2), ("allreduce", P2, Y2, g)]
        ranks.append(dict(X=X, P1=P1, P2=P2, Y1=Y1, Y2=Y2, chain=w4.Chain(ops, M, sms=sms)))
    streams = [torch.cuda.Stream() for _ in range(T)]
    for rep in range(3):   # new inputs every run: stale flags or partials would show
        for r, rk in enumerate(ranks):
            synth.gpu(12 + rep, 300 + r, synth.ACT, M, Kr, out=rk["X"])
            rk["Y1"].fill_(float("nan"))
            rk["Y2"].fill_(float("nan"))
        torch.cuda.synchronize()
        for rk, st in zip(ranks, streams):
            rk["chain"](st)
        torch.cuda.synchronize()
        for stage, (P, Y, Wm, Xs) in enumerate([("P1", "Y1", Wa, [rk["X"] for rk in ranks]),
                                                 ("P2", "Y2", Wb, [ranks[0]["Y1"]] * T)]):
            parts = [rk[P] for rk in ranks]
            want = _fp32_rank_sum(parts)
            for r, rk in enumerate(ranks):
                assert np.array_equal(_u16(rk[Y]), want), f"rep {rep} {Y} rank {r}: not the fp32 rank-order sum"
            ref = oracle.allreduce(np.stack([_u16(p) for p in parts]))
            d = np.abs(_f64(ranks[0][Y]) - ref.view(np.float16).astype(np.float64))
            ulp = np.spacing(np.abs(ref.view(np.float16))).astype(np.float64)
            assert np.all(d <= ulp), f"rep {rep} {Y}: more than 1 ulp from the oracle sum"
            if rep == 0:   # each partial is the rank's shard GEMM (oracle, GEMM tolerance)
                for r in range(T):
                    g_ref = _oracle_gemm(Xs[r], Wm[r], mode)
                    y = _f64(parts[r])
                    assert np.all(np.abs(y - g_ref) <= 1e-2 * (1 + np.abs(g_ref))), f"{P} rank {r}"


@pytest.mark.timeout(300)
def test_allreduce_result_feeds_the_next_op_in_order():
    """An op that reads an ALLREDUCE output must see the reduced values (RAW through the reduced tiles'
    ready flags): a SiLU*mul on the reduced [gate | up] equals w4a16_silu_mul applied afterwards to the same
    tensor, and a GEMM on that output equals the same GEMM launched on its own."""
    import paper_2505_22179_b200 as w4
    T, M, F = 2, 8, 1024
    sms = torch.cuda.get_device_properties(0).multi_processor_count // T
    Kr = 128 * ((sms + 2 * F // 128 - 1) // (2 * F // 128))
    f16 = dict(dtype=torch.float16, device="cuda")
    groups = w4.PeerGroup.simulated(T, 1 << 20, flag_slots=2, device="cuda")
    ranks = []
    for r, g in enumerate(groups):
        pl = w4.pack_linear(synth.gpu(21, 400 + r, synth.WEIGHT, Kr, 2 * F))
        pl2 = w4.pack_linear(synth.gpu(21, 600 + r, synth.WEIGHT, 2 * F, 2 * F))
        X = synth.gpu(21, 500 + r, synth.ACT, M, Kr)
        P = g.alloc(M, 2 * F)
        GU, act = torch.empty((M, 2 * F), **f16), torch.empty((M, F), **f16)
        P2 = g.alloc(M, 2 * F)
        out = torch.empty((M, 2 * F), **f16)
        # the second ALLREDUCE (of a GEMM on GU) keeps the alternating-partials rule satisfied
        ops = [("gemm", X, pl, P), ("allreduce", P, GU, g), ("silu_mul", GU, act), ("gemm", GU, pl2, P2),
               ("allreduce", P2, out, g)]
        ranks.append(dict(GU=GU, act=act, out=out, P2=P2, pl2=pl2, chain=w4.Chain(ops, M, sms=sms)))
    streams = [torch.cuda.Stream() for _ in range(T)]
    for rk, st in zip(ranks, streams):
        rk["chain"](st)
    torch.cuda.synchronize()
    want_out = _fp32_rank_sum([rk["P2"] for rk in ranks])
    for rk in ranks:
        want = torch.empty_like(rk["act"])
        w4.w4a16_silu_mul(rk["GU"], want)
        P2 = torch.empty_like(rk["P2"])
        ws = w4.alloc_workspace(M, [(2 * F, 2 * F)])
        rk["pl2"](rk["GU"], P2, ws)
        torch.cuda.synchronize()
        assert np.array_equal(_u16(rk["act"]), _u16(want))
        assert np.array_equal(_u16(rk["GU"]), _u16(ranks[0]["GU"]))
        # (the chain runs on half the SMs: another stream-K split, so equal up to fp32 rounding, not bitwise)
        assert torch.all((rk["P2"].float() - P2.float()).abs() <= 1e-3 * (1 + P2.float().abs())), \
            "GEMM on the reduced output != the same GEMM alone"
        assert np.array_equal(_u16(rk["out"]), want_out)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("M", [1, 8, 16])
def test_chain_allreduce_nvls_world1(M):
    """The NVLS path (PeerGroup.mc: a multicast object, tile counters bumped with multimem.red, tiles reduced
    with multimem.ld_reduce) on this box's one GPU (world 1): over repeated runs the chain's reduced outputs
    equal the fp32 rank-order definition (at world 1: the partial itself) bit for bit, the partials equal the
    same chain over a simulated (peer-load) group, and a GEMM reading the reduced output sees it."""
    import paper_2505_22179_b200 as w4
    if not w4.PeerGroup.mc_supported():
        pytest.skip("no multicast / fabric-handle support on this device")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    H = 1024
    Kr = 128 * -(-sms // (H // 128))
    f16 = dict(dtype=torch.float16, device="cuda")
    pa = w4.pack_linear(synth.gpu(31, 1, synth.WEIGHT, Kr, H))
    pb = w4.pack_linear(synth.gpu(31, 2, synth.WEIGHT, H, Kr))
    X = torch.empty((M, Kr), **f16)
    outs = {}
    try:
        w4.PeerGroup.mc(1 << 21, 4).close()
    except w4.W4A16Error as e:   # e.g. a GPU partition whose driver refuses cuMulticastCreate
        pytest.skip(f"multicast object creation not available here: {e}")
    for kind in ("nvls", "peer"):
        g = w4.PeerGroup.mc(1 << 21, 4) if kind == "nvls" else w4.PeerGroup.simulated(1, 1 << 21, 4, device="cuda")[0]
        assert g.kind == kind
        P1, P2 = g.alloc(M, H), g.alloc(M, Kr)
        Y1, Y2 = torch.empty((M, H), **f16), torch.empty((M, Kr), **f16)
        ch = w4.Chain([("gemm", X, pa, P1), ("allreduce", P1, Y1, g), ("gemm", Y1, pb, P2), ("allreduce", P2, Y2, g)], M)
        res = []
        for rep in range(3):   # fresh inputs every run: stale counters or partials would show
            synth.gpu(32 + rep, 7, synth.ACT, M, Kr, out=X)
            Y1.fill_(float("nan"))
            Y2.fill_(float("nan"))
            ch()
            torch.cuda.synchronize()
            assert np.array_equal(_u16(Y1), _u16(P1)), f"{kind} rep {rep}: Y1 != P1 (world 1)"
            assert np.array_equal(_u16(Y2), _u16(P2)), f"{kind} rep {rep}: Y2 != P2 (world 1)"
            res.append((_u16(P1).copy(), _u16(P2).copy()))
        outs[kind] = res
        del ch
        g.close()
    for rep in range(3):
        assert np.array_equal(outs["nvls"][rep][0], outs["peer"][rep][0])
        assert np.array_equal(outs["nvls"][rep][1], outs["peer"][rep][1])


@pytest.mark.timeout(600)
@pytest.mark.parametrize("M", [1, 8, 16])
def test_tp2_fused_stack_matches_tp1(M):
    """tp.py with allreduce="fused": two simulated ranks of a 2-layer stack (each one chain per forward with
    ALLREDUCE ops) give identical reduced outputs on both ranks, within the GEMM tolerance of the tp = 1
    stack built from the same full weights and inputs."""
    import paper_2505_22179_b200 as w4
    from paper_2505_22179_b200 import tp
    # one layer: with the real data flow, a second layer would compare values that already differ by the tp
    # rounding of layer 1 (fp16 partials per rank, reading R20) amplified through four more GEMMs; the protocol
    # (two ALLREDUCE slots per run, repeated runs, both ranks bit-identical) is exercised all the same
    T, layers = 2, 1
    dims = tp.ModelDims("tiny", hidden=2048, ffn=4096, n_q=16, n_kv=4, head=128, layers=layers)
    sms = torch.cuda.get_device_properties(0).multi_processor_count // T
    full = {}

    def make(rank, t):
        def mk(l, name, K, N, out):
            if (l, name) not in full:
                Kf, Nf = tp.shard_plan(dims, 1, 0)[name]["full"]
                W = synth.gpu(31, 1000 + 10 * l + tp.MATRICES.index(name), synth.WEIGHT, Kf, Nf)
                # ~unit gain (std of the generated weights incl. their outlier groups): O(1) activations through
                # the dependent stack, so the absolute part of the tolerance stays meaningful in layer 2
                full[(l, name)] = W.mul_(1.0 / (float(W.float().std()) * Kf ** 0.5))
            out.copy_(tp.shard_of(full[(l, name)], tp.shard_plan(dims, t, rank)[name]))
        return mk

    ref = tp.VerifyStack(dims, layers, 16, make(0, 1), device="cuda")
    groups = w4.PeerGroup.simulated(T, 1 << 22, 2 * layers, device="cuda")
    ranks = [tp.VerifyStack(dims, layers, 16, make(r, T), tp_size=T, tp_rank=r, allreduce="fused",
                            peer_group=groups[r], chain_sms=sms, device="cuda") for r in range(T)]
    x_in = synth.gpu(32, 1, synth.ACT, 16, dims.hidden)
    for st in [ref] + ranks:
        st.x_in.copy_(x_in)
    ref.forward(M)
    streams = [torch.cuda.Stream() for _ in range(T)]
    for rep in range(2):
        for st in ranks:
            st.y_o_red.fill_(float("nan"))
            st.y_down_red.fill_(float("nan"))
        torch.cuda.synchronize()
        for st, s in zip(ranks, streams):
            with torch.cuda.stream(s):
                st.forward(M, stream=s)
        torch.cuda.synchronize()
        for name in ("y_o_red", "y_down_red"):
            a = [getattr(st, name)[:M] for st in ranks]
            assert torch.equal(a[0].view(torch.int16), a[1].view(torch.int16)), name
            want = _f64(getattr(ref, name)[:M])
            got = _f64(a[0])
            assert np.all(np.abs(got - want) <= 1e-2 * (1 + np.abs(want))), f"{name} rep {rep}"
        assert ranks[0].launches_per_forward(M) == 2
