"""W4A8 variant (include/w4a16.h w4a8_*; reading R21): the GPU activation quantisation is
bit-exact with the oracle (codes, fp32 scales, group sums — integers decided in fp32 on both sides), and the
W4A8 GEMM on the SYM blob matches the oracle's exact-integer definition within the fp32-epilogue / fp16
output tolerance, over ragged token counts and several tiles."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
SYM = 1


def _w4():
    import paper_2505_22179_b200 as w4
    return w4


def _quant_gpu(X):
    w4 = _w4()
    M, K = X.shape
    Xq = torch.empty(M, K, dtype=torch.int8, device="cuda")
    sx = torch.empty(M, dtype=torch.float32, device="cuda")
    xs = torch.empty(M, K // 128, dtype=torch.int32, device="cuda")
    w4.w4a8_quantize_act(X, Xq, sx, xs)
    torch.cuda.synchronize()
    return Xq, sx, xs


@pytest.mark.parametrize("M,K", [(1, 128), (7, 1024), (16, 8192), (64, 4096)])
def test_act_quant_bit_exact(M, K):
    X = synth.gpu(41, M * 10 + K, synth.ACT, M, K)
    if M > 1:
        X[1].zero_()                     # zero row: codes 0, scale 0
    if M > 2:
        X[2, :8] = torch.tensor([127.0, 0.5, 1.5, 2.5, -0.5, -2.5, 3.5, -127.0], dtype=torch.float16)
        X[2, 8:] = 0                     # inv = 1 exactly: round-half-even ties decided by the kernel
    Xq, sx, xs = _quant_gpu(X)
    q_ref, s_ref, xs_ref = oracle.quantize_act_int8(X.view(torch.int16).cpu().numpy().view(np.uint16))
    assert np.array_equal(Xq.cpu().numpy(), q_ref)
    assert np.array_equal(sx.cpu().numpy().view(np.uint32), s_ref.view(np.uint32))
    assert np.array_equal(xs.cpu().numpy(), xs_ref)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("impl", [0, 1, 2])
@pytest.mark.parametrize("M", [1, 5, 8, 16, 33, 64])
@pytest.mark.parametrize("K,N", [(1024, 1280), (4096, 2560)])
def test_w4a8_gemm_vs_oracle(M, K, N, impl):
    # impl: 0 = auto, 1 = the family-A pipeline (M <= 16: int8 codes (q - 8) * 16, mma m16n8k32 s8), 2 = round 1
    if impl == 1 and M > 16:
        pytest.skip("the family-A W4A8 path serves M <= 16")
    w4 = _w4()
    W = synth.host(42, K + N, synth.WEIGHT, K, N)
    Wd = torch.from_numpy(W.view(np.int16)).cuda().view(torch.float16)
    pl = w4.pack_linear(Wd, mode=w4.W4A16_SYM)
    X = synth.gpu(43, M + K, synth.ACT, M, K)
    Xq, sx, xs = _quant_gpu(X)
    ws = torch.zeros(w4.w4a8_workspace_bytes(M, K, N), dtype=torch.uint8, device="cuda")
    Y = torch.full((M, N), float("nan"), dtype=torch.float16, device="cuda")
    w4.w4a8_gemm(Xq, sx, xs, pl.packed, Y, ws, impl=impl)
    torch.cuda.synchronize()
    # the oracle quantises the HOST activations itself; the GPU's codes / scales / group sums must equal them
    # bit for bit, and only the oracle's own values feed the oracle GEMM
    q_ref, s_ref, xs_ref = oracle.quantize_act_int8(X.view(torch.int16).cpu().numpy().view(np.uint16))
    assert np.array_equal(Xq.cpu().numpy(), q_ref)
    assert np.array_equal(sx.cpu().numpy().view(np.uint32), s_ref.view(np.uint32))
    assert np.array_equal(xs.cpu().numpy(), xs_ref)
    codes, sc, _, _ = oracle.quantize(W, 128, SYM)
    ref = oracle.gemm_w4a8(q_ref, s_ref, codes, sc)
    y = Y.float().cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(y))
    assert np.all(np.abs(y - ref) <= 1e-3 * (1 + np.abs(ref))), np.abs(y - ref).max()
    # deterministic: a second run gives the same bits
    Y2 = torch.empty_like(Y)
    w4.w4a8_gemm(Xq, sx, xs, pl.packed, Y2, ws, impl=impl)
    torch.cuda.synchronize()
    assert torch.equal(Y.view(torch.int16), Y2.view(torch.int16))


def test_w4a8_rejects_bad_arguments():
    w4 = _w4()
    X = torch.zeros(4, 200, dtype=torch.float16, device="cuda")     # K % 128 != 0
    with pytest.raises(w4.W4A16Error):
        w4.w4a8_quantize_act(X, torch.empty(4, 200, dtype=torch.int8, device="cuda"),
                             torch.empty(4, dtype=torch.float32, device="cuda"),
                             torch.empty(4, 1, dtype=torch.int32, device="cuda"))
