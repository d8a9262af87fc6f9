"""The C-ABI library loads, exports every symbol include/w4a16.h declares, and rejects bad arguments on the
host before touching the GPU (-m "not gpu": no compute call is made without a GPU)."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "w4a16.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return re.findall(r"^\s*(?:int|size_t|const char\s*\*)\s+(\w+)\s*\(", src, flags=re.M)


def test_header_declares_the_abi():
    names = declared_functions()
    for required in ("w4a16_pack", "w4a16_unpack", "w4a16_gemm", "w4a16_gemm_workspace_bytes", "verify_accept",
                     "w4a16_status_string"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2505_22179_b200 import _lib
    names = declared_functions()
    assert set(names) == set(_lib.ABI_SYMBOLS)
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), n


def test_status_strings():
    from paper_2505_22179_b200 import w4a16_status_string
    assert w4a16_status_string(0) == "W4A16_OK"
    for s in (-1, -2, -3, -4, -5):
        assert w4a16_status_string(s).startswith("W4A16_ERR")
    assert "unknown" in w4a16_status_string(17)


def test_host_validation_before_any_cuda_call():
    from paper_2505_22179_b200._lib import lib
    A = 0x10000  # a 16-byte-aligned fake device address: validation must reject before dereferencing
    # w4a16_gemm(X, packed, Y, M, K, N, group, mode, ws, ws_bytes, stream)
    assert lib.w4a16_gemm(None, A, A, 8, 4096, 4096, 128, 0, A, 1 << 20, None) == -1
    assert lib.w4a16_gemm(A, None, A, 8, 4096, 4096, 128, 0, A, 1 << 20, None) == -1
    assert lib.w4a16_gemm(A, A, A, 8, 4096, 4096, 64, 0, A, 1 << 20, None) == -1       # group must be 128
    assert lib.w4a16_gemm(A, A, A, 8, 4000, 4096, 128, 0, A, 1 << 20, None) == -2
    assert lib.w4a16_gemm(A, A, A, 8, 4096, 4100, 128, 0, A, 1 << 20, None) == -2
    assert lib.w4a16_gemm(A, A, A, 0, 4096, 4096, 128, 0, A, 1 << 20, None) == -2
    assert lib.w4a16_gemm(A, A, A, 65, 4096, 4096, 128, 0, A, 1 << 20, None) == -2
    assert lib.w4a16_gemm(A + 2, A, A, 8, 4096, 4096, 128, 0, A, 1 << 20, None) == -3
    assert lib.w4a16_gemm(A, A, A, 8, 4096, 4096, 128, 7, A, 1 << 20, None) == -1     # bad mode
    assert lib.w4a16_gemm_ex(A, A, A, 8, 4096, 4096, 128, 0, A, 1 << 20, 5, None) in (-1, -5)  # bad family
    assert lib.w4a16_pack(A, 4096, 4096, 128, 0, None, None, None) == -1
    assert lib.w4a16_pack(A, 100, 4096, 128, 0, A, None, None) == -2
    assert lib.w4a16_unpack(A, 4096, 4096, 128, 1, A + 8, None) == -3
    assert lib.w4a16_packed_bytes(4096, 4096, 128, 0) == 32 * 32 * 8704
    assert lib.w4a16_packed_bytes(4096, 4096, 128, 1) == 32 * 32 * 8448
    assert lib.w4a16_packed_bytes(4096, 4000, 128, 0) == 0
    assert lib.verify_accept(A, A, A, 0, A, None) == -2
    assert lib.verify_accept(A, A, A, 1025, A, None) == -2
    assert lib.verify_accept(None, A, A, 8, A, None) == -1
    assert lib.w4a16_gemm_workspace_bytes(8, 4000, 4096, 128) == 0
    # W4A8: the GEMM reads Xq and the blob with 16-byte copies, so 4- or 8-byte alignment is rejected on the host
    # w4a8_quantize_act(X, M, K, Xq, sx, xsum, stream); w4a8_gemm(Xq, sx, xsum, packed, Y, M, K, N, ws, ws_bytes, stream)
    assert lib.w4a8_quantize_act(A, 8, 4096, A + 4, A, A, None) == -3
    assert lib.w4a8_quantize_act(A, 8, 4096, A, A + 2, A, None) == -3
    assert lib.w4a8_quantize_act(A, 8, 4096, A, A, A + 1, None) == -3
    for xq, pk, sx, xs in ((A + 4, A, A, A), (A + 8, A, A, A), (A, A + 4, A, A), (A, A + 8, A, A), (A, A, A + 2, A),
                           (A, A, A, A + 2)):
        assert lib.w4a8_gemm(xq, sx, xs, pk, A, 8, 4096, 4096, A, 1 << 30, None) == -3


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    # valid arguments on a machine without a GPU: the library reports a CUDA failure, it never computes on CPU
    from paper_2505_22179_b200._lib import lib
    A = 0x10000
    assert lib.w4a16_gemm(A, A, A, 8, 4096, 4096, 128, 0, A, 1 << 30, None) == -5
    assert lib.w4a16_gemm_workspace_bytes(8, 4096, 4096, 128) == 0


def test_product_never_touches_the_oracle():
    # the product path (package + CUDA sources) shares no code with oracle/ and never imports it
    pkg = os.path.join(ROOT, "paper_2505_22179_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("w4a16_oracle", "import oracle", "from oracle", "orc_", "libw4a16_oracle"):
                    assert bad not in txt, (f, bad)
    hdr = open(HEADER).read()
    assert "w4a16_oracle" not in hdr and "orc_" not in hdr
