"""Tree-masked verify attention and KV compaction (include/w4a16.h w4a16_tree_attention,
w4a16_kv_compact) against the CPU oracle.

Tolerance (derived): the kernel rounds the softmax probabilities to fp16 for the P.V MMA
(relative error <= 2^-11 per weight) and the output to fp16 (2^-11 |O|), everything else in fp32; with
|v| = O(1) this stays below 4e-3 * (1 + |O|). Masking is checked structurally as well: perturbing the
keys/values of tree rows that are not ancestors of a row leaves that row's output bit-identical. The KV
compaction moves bytes and must be bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL = 4e-3


def _w4():
    import paper_2505_22179_b200 as w4
    return w4


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _gpu_attn(Q, K, V, par):
    w4 = _w4()
    M, Hq, D = Q.shape
    Lt, Hkv, _ = K.shape
    Qd, Kd, Vd = _t(Q), _t(K), _t(V)
    O = torch.full((M, Hq, D), float("nan"), dtype=torch.float16, device="cuda")
    ws = torch.zeros(w4.w4a16_tree_attention_workspace_bytes(M, Lt - M, Hq, Hkv, D), dtype=torch.uint8, device="cuda")
    w4.w4a16_tree_attention(Qd, Kd, Vd, _t(np.asarray(par, dtype=np.int32)), O, ws)
    torch.cuda.synchronize()
    return O.float().cpu().numpy().astype(np.float64)


def _inputs(seed, M, L, Hq, Hkv, D=128):
    rng = np.random.default_rng(seed)
    Q = (0.5 * rng.standard_normal((M, Hq, D))).astype(np.float16)
    K = (0.5 * rng.standard_normal((L + M, Hkv, D))).astype(np.float16)
    V = rng.standard_normal((L + M, Hkv, D)).astype(np.float16)
    return Q, K, V


@pytest.mark.parametrize("M,L,Hq,Hkv,kind", [(1, 0, 8, 1, "seq"), (1, 37, 8, 8, "seq"), (7, 100, 8, 2, "seq"),
                                             (8, 64, 16, 2, "tree"), (16, 300, 16, 2, "tree"), (49, 513, 64, 8, "tree"),
                                             (61, 1000, 64, 8, "tree"), (64, 130, 8, 1, "seq")])
def test_tree_attention_vs_oracle(M, L, Hq, Hkv, kind):
    Q, K, V = _inputs(M * 1000 + L, M, L, Hq, Hkv)
    if kind == "seq":
        par = np.arange(-1, M - 1, dtype=np.int32)
    else:
        _, par = synth.eagle_tree(np.random.default_rng(M + L), M - 1, 6)
        par = np.asarray(par, dtype=np.int32)
    ref = oracle.tree_attention(Q, K, V, par)
    got = _gpu_attn(Q, K, V, par)
    err = np.abs(got - ref)
    assert np.all(err <= TOL * (1 + np.abs(ref))), f"max err {err.max():.3g}"


def test_tree_attention_bench_config_and_workspace_reuse():
    # the bench's configuration (70B head layout, L = 2048, M = 8 and 61: many splits merged in-kernel), then a
    # small problem (one split, no merge) and the big one again on the SAME workspace: the split-merge counters
    # in its header must come back to zero after every call (include/w4a16.h)
    w4 = _w4()
    Hq, Hkv, D = 64, 8, 128
    cases = [(8, 2048), (61, 2048), (3, 20), (8, 2048)]
    nbytes = max(w4.w4a16_tree_attention_workspace_bytes(M, L, Hq, Hkv, D) for M, L in cases)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    for M, L in cases:
        Q, K, V = _inputs(M + 7 * L, M, L, Hq, Hkv)
        _, par = synth.eagle_tree(np.random.default_rng(M), M - 1, 6)
        par = np.asarray(par, dtype=np.int32)
        O = torch.full((M, Hq, D), float("nan"), dtype=torch.float16, device="cuda")
        w4.w4a16_tree_attention(_t(Q), _t(K), _t(V), _t(par), O, ws)
        torch.cuda.synchronize()
        got = O.float().cpu().numpy().astype(np.float64)
        ref = oracle.tree_attention(Q, K, V, par)
        err = np.abs(got - ref)
        assert np.all(err <= TOL * (1 + np.abs(ref))), f"M={M} L={L}: max err {err.max():.3g}"
        assert int(ws[:65536].view(torch.int32)[0::32].abs().sum()) == 0, "split-merge counters not re-armed"


def test_tree_attention_masks_non_ancestors_exactly():
    M, L, Hq, Hkv = 12, 50, 8, 2
    Q, K, V = _inputs(7, M, L, Hq, Hkv)
    par = np.array([-1, 0, 0, 1, 1, 2, 3, 3, 5, 8, 0, 10], dtype=np.int32)
    base = _gpu_attn(Q, K, V, par)
    rng = np.random.default_rng(8)
    for i in (4, 9, 11):
        anc, a = set(), i
        while a != -1:
            anc.add(a)
            a = int(par[a])
        others = [j for j in range(M) if j not in anc]
        K2, V2 = K.copy(), V.copy()
        K2[[L + j for j in others]] = rng.standard_normal((len(others), Hkv, 128)).astype(np.float16)
        V2[[L + j for j in others]] = rng.standard_normal((len(others), Hkv, 128)).astype(np.float16)
        pert = _gpu_attn(Q, K2, V2, par)
        assert np.array_equal(pert[i], base[i]), f"row {i} sees a non-ancestor"


def test_kv_compact_bit_exact_after_gpu_accept():
    w4 = _w4()
    L, Hkv, D = 33, 8, 128
    tok = [100, 11, 12, 21, 22, 23, 31, 32]
    par = [-1, 0, 0, 1, 1, 2, 3, 5]
    am = [12, 99, 23, 31, 99, 32, 99, 40]
    M = len(tok)
    _, K, V = _inputs(9, M, L, 8, Hkv)
    out = torch.empty(3 + M, dtype=torch.int32, device="cuda")
    w4.verify_accept(_t(np.array(tok, dtype=np.int32)), _t(np.array(par, dtype=np.int32)),
                     _t(np.array(am, dtype=np.int32)), out)
    Kd, Vd = _t(K), _t(V)
    w4.w4a16_kv_compact(Kd, Vd, L, out)
    torch.cuda.synchronize()
    Kr, Vr = oracle.kv_compact(K, V, L, oracle.accept(tok, par, am)[4])
    assert np.array_equal(Kd.cpu().numpy().view(np.uint16), Kr.view(np.uint16))
    assert np.array_equal(Vd.cpu().numpy().view(np.uint16), Vr.view(np.uint16))


@pytest.mark.timeout(60)
def test_tree_attention_malformed_parents_do_not_hang():
    # a cycle (3 -> 5 -> 3), a self-loop (6 -> 6) and an out-of-range parent (9 -> 40 >= M): the kernel must
    # finish, and a row whose ancestry walk meets an invalid link sees the prefix and itself only
    # (include/w4a16.h) — which the oracle computes for parents[row] = -1
    M, L, Hq, Hkv = 12, 50, 8, 2
    Q, K, V = _inputs(77, M, L, Hq, Hkv)
    par = np.arange(-1, M - 1, dtype=np.int32)
    par[3], par[5], par[6], par[9] = 5, 3, 6, 40
    par[10] = 9                                   # valid link into an invalid row: invalid too
    got = _gpu_attn(Q, K, V, par)

    def walk_ok(x):
        while x >= 0:
            px = int(par[x])
            if px < -1 or px >= x:
                return False
            x = px
        return True

    bad = [x for x in range(M) if not walk_ok(x)]
    assert bad == [3, 4, 5, 6, 7, 8, 9, 10, 11]
    # valid rows 0..2 (a chain): the oracle on that sub-tree (their keys sit at L..L+2)
    ref = oracle.tree_attention(Q[:3], K[:L + 3], V[:L + 3], par[:3])
    assert np.all(np.abs(got[:3] - ref) <= TOL * (1 + np.abs(ref)))
    # each invalid row: the oracle on a one-row problem over the prefix plus that row's own key / value
    for x in bad:
        Kx = np.concatenate([K[:L], K[L + x:L + x + 1]])
        Vx = np.concatenate([V[:L], V[L + x:L + x + 1]])
        ref = oracle.tree_attention(Q[x:x + 1], Kx, Vx, np.array([-1], dtype=np.int32))
        assert np.all(np.abs(got[x:x + 1] - ref) <= TOL * (1 + np.abs(ref))), x


def test_tree_attention_cuda_graph_replays():
    # the bench replays the cooperative launch inside a CUDA graph: every replay must leave the split-merge
    # counters re-armed and give the same (bit-identical) output as an eager call
    w4 = _w4()
    M, L, Hq, Hkv, D = 8, 2048, 64, 8, 128
    Q, K, V = _inputs(4242, M, L, Hq, Hkv)
    _, par = synth.eagle_tree(np.random.default_rng(5), M - 1, 6)
    Qd, Kd, Vd, pd = _t(Q), _t(K), _t(V), _t(np.asarray(par, dtype=np.int32))
    ws = torch.zeros(w4.w4a16_tree_attention_workspace_bytes(M, L, Hq, Hkv, D), dtype=torch.uint8, device="cuda")
    O_eager = torch.empty(M, Hq, D, dtype=torch.float16, device="cuda")
    w4.w4a16_tree_attention(Qd, Kd, Vd, pd, O_eager, ws)
    O = torch.full((M, Hq, D), float("nan"), dtype=torch.float16, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        w4.w4a16_tree_attention(Qd, Kd, Vd, pd, O, ws, stream=s)
    for _ in range(3):
        O.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(O.view(torch.int16), O_eager.view(torch.int16))
        assert int(ws[:65536].view(torch.int32)[0::32].abs().sum()) == 0
