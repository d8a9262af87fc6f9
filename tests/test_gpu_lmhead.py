"""LM head + greedy argmax (include/w4a16.h w4a16_lmhead_argmax) against the CPU oracle.

The oracle computes every logit in fp64 and takes the first maximum. The GPU decides on fp32 sums
(reading R19): the kernel accumulates each logit as K/16 sequential fp32 additions of 16-product MMA results,
so its error is bounded by B[m][v] = (K/16 + 16) * 2^-23 * sum_k |H[m][k] W[v][k]| (u = 2^-23 also covers a
truncating accumulator; the products are exact). Where several ids lie within those bounds of the maximum
either may win; so the GPU's pick v must satisfy logit[v] >= logit[v*] - B[v*] - B[v], its reported logit
must be within B[v] of the fp64 logit, and wherever the fp64 best v* beats EVERY other id by more than the
sum of their bounds the ids must be identical. Exact ties (identical weight rows) give identical fp32 sums,
so the lowest id must win bit-exactly."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1


def _w4():
    import paper_2505_22179_b200 as w4
    return w4


def _gpu(H_u16, W_u16):
    w4 = _w4()
    M, K = H_u16.shape
    V = W_u16.shape[0]
    H = torch.from_numpy(H_u16.view(np.int16)).cuda().view(torch.float16)
    W = torch.from_numpy(W_u16.view(np.int16)).cuda().view(torch.float16)
    idx = torch.full((M,), -7, dtype=torch.int32, device="cuda")
    val = torch.full((M,), float("nan"), dtype=torch.float32, device="cuda")
    ws = w4.alloc_lmhead_workspace(M, K, V)
    w4.w4a16_lmhead_argmax(H, W, idx, ws, out_max=val)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), val.cpu().numpy().astype(np.float64)


def _check(H_u16, W_u16, gi, gv):
    idx, val, lg = oracle.lmhead_argmax(H_u16, W_u16, nthreads=NPROC, want_logits=True)
    M, K = H_u16.shape
    rows = np.arange(M)
    habs = np.abs(H_u16.view(np.float16).astype(np.float64))
    wabs = np.abs(W_u16.view(np.float16).astype(np.float64))
    B = (K / 16 + 16) * 2.0 ** -23 * (habs @ wabs.T)          # fp32 accumulation bound per logit
    assert np.all((gi >= 0) & (gi < W_u16.shape[0]))
    assert np.all(lg[rows, gi] >= val - B[rows, idx] - B[rows, gi]), "GPU argmax is not a maximiser within the bound"
    assert np.all(np.abs(gv - lg[rows, gi]) <= B[rows, gi]), "reported max logit off"
    others = lg + B
    others[rows, idx] = -np.inf
    clear = (val - B[rows, idx]) > others.max(axis=1)        # v* beats every other id beyond both bounds
    assert np.array_equal(gi[clear], idx[clear])
    return clear.mean()


@pytest.mark.parametrize("M,K,V", [(1, 128, 128), (5, 1024, 2048), (8, 4096, 6400), (13, 2048, 4096), (40, 512, 3072),
                                   (64, 1024, 1280)])
def test_lmhead_argmax_vs_oracle(M, K, V):
    H = synth.host(5 + M, 31, synth.ACT, M, K)
    W = synth.host(6 + V, 32, synth.WEIGHT, V, K)
    gi, gv = _gpu(H, W)
    _check(H, W, gi, gv)


def test_lmhead_argmax_planted_and_ties():
    rng = np.random.default_rng(3)
    M, K, V = 9, 1024, 3840
    H = synth.host(8, 33, synth.ACT, M, K)
    W = synth.host(9, 34, synth.WEIGHT, V, K).view(np.float16).copy()
    plant = rng.choice(V, size=M, replace=False)
    for m, v in enumerate(plant):
        W[v] = (H[m].view(np.float16).astype(np.float32) * 0.25).astype(np.float16)
    gi, _ = _gpu(H, W.view(np.uint16))
    assert np.array_equal(gi, plant)
    # exact ties: copy each planted winner to two other ids -> the lowest of the three ids wins
    W2 = W.copy()
    used, want = set(int(v) for v in plant), []
    for m, v in enumerate(plant):
        ids = [int(v)]
        for cand in ((v * 7 + 3) % V, (v + V // 2) % V):
            c = int(cand)
            while c in used:
                c = (c + 1) % V
            used.add(c)
            W2[c] = W[v]
            ids.append(c)
        want.append(min(ids))
    gi2, _ = _gpu(H, W2.view(np.uint16))
    ref, _ = oracle.lmhead_argmax(H, W2.view(np.uint16), nthreads=NPROC)
    assert np.array_equal(gi2, np.array(want))
    assert np.array_equal(gi2, ref)


@pytest.mark.timeout(600)
def test_lmhead_argmax_llama3_70b_full_size():
    # BASELINE.json config 4 shape of the head: K = 8192, V = 128256 (Llama-3 vocabulary), verify width 8
    M, K, V = 8, 8192, 128256
    w4 = _w4()
    W = synth.gpu(13, 35, synth.WEIGHT, V, K)
    H = synth.gpu(13, 36, synth.ACT, M, K)
    idx = torch.empty(M, dtype=torch.int32, device="cuda")
    val = torch.empty(M, dtype=torch.float32, device="cuda")
    ws = w4.alloc_lmhead_workspace(M, K, V)
    for _ in range(2):   # the second call checks the workspace re-arming
        w4.w4a16_lmhead_argmax(H, W, idx, ws, out_max=val)
    torch.cuda.synchronize()
    Hn = synth.host(13, 36, synth.ACT, M, K)
    Wn = synth.host(13, 35, synth.WEIGHT, V, K)
    _check(Hn, Wn, idx.cpu().numpy(), val.cpu().numpy().astype(np.float64))


def test_lmhead_argmax_graph_capture_feeds_verify_accept():
    # the head's argmax is verify_accept's target_argmax input; both captured in one CUDA graph
    w4 = _w4()
    M, K, V = 7, 1024, 2560
    H = synth.gpu(1, 37, synth.ACT, M, K)
    W = synth.gpu(1, 38, synth.WEIGHT, V, K)
    am = torch.empty(M, dtype=torch.int32, device="cuda")
    ws = w4.alloc_lmhead_workspace(M, K, V)
    w4.w4a16_lmhead_argmax(H, W, am, ws)
    torch.cuda.synchronize()
    ref_am = am.cpu().numpy().copy()
    # a sequence draft whose first 3 tokens agree with the target's greedy choices
    toks = np.array([5] + [int(ref_am[i]) for i in range(3)] + [int(ref_am[3]) + 1, 0, 0][:M - 4], dtype=np.int32)
    par = np.arange(-1, M - 1, dtype=np.int32)
    t = torch.from_numpy(toks).cuda()
    p = torch.from_numpy(par).cuda()
    out = torch.empty(3 + M, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        w4.w4a16_lmhead_argmax(H, W, am, ws, stream=s)
        w4.verify_accept(t, p, am, out, stream=s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        w4.w4a16_lmhead_argmax(H, W, am, ws, stream=s)
        w4.verify_accept(t, p, am, out, stream=s)
    am.fill_(-1)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(am.cpu().numpy(), ref_am)
    assert np.array_equal(out.cpu().numpy(), oracle.accept(toks, par, ref_am)[4])
    assert int(out[0]) == 3
