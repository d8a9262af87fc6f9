"""Same-name Python binding of the C ABI (include/w4a16.h) over torch tensors.

Each function checks dtypes/devices, passes raw device pointers and the current CUDA stream to
libw4a16.so, and raises W4A16Error on a non-zero status. Nothing here computes any part of the path.
"""
from dataclasses import dataclass
from typing import Optional

import torch

from ._lib import (  # noqa: F401
    lib, check, status_string, W4A16Error,
    W4A16_ASYM, W4A16_SYM, W4A16_GROUP, W4A16_MAX_M, W4A16_MAX_TREE,
    W4A16_DEV_OK, W4A16_DEV_NONFINITE, W4A16_DEV_BAD_TREE,
    W4A16_FAMILY_AUTO, W4A16_FAMILY_MMA_SYNC, W4A16_FAMILY_TCGEN05, W4A16_FAMILY_MMA_SYNC_S,
)


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _ptr(t: Optional[torch.Tensor], dtype=None, name="tensor") -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise W4A16Error(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise W4A16Error(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise W4A16Error(f"{name} must be contiguous")
    return t.data_ptr()


def w4a16_packed_bytes(K: int, N: int, mode=W4A16_ASYM, group=W4A16_GROUP) -> int:
    n = int(lib.w4a16_packed_bytes(K, N, group, mode))
    if n == 0:
        raise W4A16Error(f"bad packed shape K={K} N={N} mode={mode} group={group}")
    return n


def w4a16_pack(W, packed, dev_status=None, mode=W4A16_ASYM, group=W4A16_GROUP, stream=None):
    K, N = W.shape
    if packed.numel() * packed.element_size() < w4a16_packed_bytes(K, N, mode, group):
        raise W4A16Error("packed buffer too small")
    st = lib.w4a16_pack(_ptr(W, torch.float16, "W"), K, N, group, mode, _ptr(packed, None, "packed"),
                        _ptr(dev_status, torch.int32, "dev_status"), _stream(stream))
    check(st, "w4a16_pack")


def w4a16_unpack(packed, W_hat, mode=W4A16_ASYM, group=W4A16_GROUP, stream=None):
    K, N = W_hat.shape
    st = lib.w4a16_unpack(_ptr(packed, None, "packed"), K, N, group, mode, _ptr(W_hat, torch.float16, "W_hat"),
                          _stream(stream))
    check(st, "w4a16_unpack")


def w4a16_gemm_workspace_bytes(M: int, K: int, N: int, group: int = W4A16_GROUP) -> int:
    return int(lib.w4a16_gemm_workspace_bytes(M, K, N, group))


def w4a16_workspace_init(workspace, stream=None):
    check(lib.w4a16_workspace_init(_ptr(workspace, None, "workspace"), workspace.numel() * workspace.element_size(),
                                   _stream(stream)), "w4a16_workspace_init")


def alloc_workspace(M_max: int, shapes, device=None) -> torch.Tensor:
    """Zero-initialised workspace big enough for every (K, N) in `shapes` at any M <= M_max."""
    need = max(w4a16_gemm_workspace_bytes(m, K, N) for K, N in shapes for m in range(1, M_max + 1))
    return torch.zeros(max(need, 256), dtype=torch.uint8, device=device or "cuda")


def w4a16_gemm(X, packed, Y, workspace, mode=W4A16_ASYM, group=W4A16_GROUP, stream=None, family=W4A16_FAMILY_AUTO):
    """Y = X . W_hat through w4a16_gemm (family AUTO) or w4a16_gemm_ex (explicit family)."""
    M, K = X.shape
    N = Y.shape[1]
    if Y.shape[0] != M:
        raise W4A16Error("Y must be [M, N]")
    args = (_ptr(X, torch.float16, "X"), _ptr(packed, None, "packed"), _ptr(Y, torch.float16, "Y"), M, K, N, group,
            mode, _ptr(workspace, None, "workspace"), workspace.numel() * workspace.element_size())
    if family == W4A16_FAMILY_AUTO:
        st = lib.w4a16_gemm(*args, _stream(stream))
    else:
        st = lib.w4a16_gemm_ex(*args, family, _stream(stream))
    check(st, "w4a16_gemm")


def verify_accept(tokens, parents, target_argmax, out, stream=None):
    n = tokens.numel()
    st = lib.verify_accept(_ptr(tokens, torch.int32, "tokens"), _ptr(parents, torch.int32, "parents"),
                           _ptr(target_argmax, torch.int32, "target_argmax"), n, _ptr(out, torch.int32, "out"),
                           _stream(stream))
    check(st, "verify_accept")


def w4a16_silu_mul(GU, out, stream=None):
    M, F2 = GU.shape
    check(lib.w4a16_silu_mul(_ptr(GU, torch.float16, "GU"), M, F2 // 2, _ptr(out, torch.float16, "out"),
                             _stream(stream)), "w4a16_silu_mul")


def w4a16_status_string(status: int) -> str:
    return status_string(status)


def w4a16_gemm_family(M: int, K: int, N: int) -> int:
    return int(lib.w4a16_gemm_family(M, K, N))


@dataclass
class PackedLinear:
    """A W4A16 linear layer resident in HBM: Y[M, N] = X[M, K] · W_hat[K, N] (packed blob, include/w4a16.h)."""
    K: int
    N: int
    mode: int
    packed: torch.Tensor

    @property
    def weight_bytes(self) -> int:
        """Algorithmic bytes streamed per GEMM (codes + scales (+ zeros)) = the blob size."""
        return self.packed.numel() * self.packed.element_size()

    def __call__(self, X, Y, workspace, stream=None, family=W4A16_FAMILY_AUTO):
        w4a16_gemm(X, self.packed, Y, workspace, self.mode, stream=stream, family=family)
        return Y


def pack_linear(W: torch.Tensor, mode=W4A16_ASYM, dev_status=None, stream=None) -> PackedLinear:
    K, N = W.shape
    packed = torch.empty(w4a16_packed_bytes(K, N, mode), dtype=torch.uint8, device=W.device)
    w4a16_pack(W, packed, dev_status, mode, stream=stream)
    return PackedLinear(K, N, mode, packed)
