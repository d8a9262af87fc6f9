"""B200-native (sm_100a) W4A16 verification hot path of arXiv 2505.22179 (HierSpec).

Python surface = the C ABI of include/w4a16.h with the same names (torch tensors in, argument
marshalling only) plus the tensor-parallel verify stack (tp.py). PyTorch supplies device memory,
streams and process groups; every step of the path runs in libw4a16.so's kernels.
"""
from .ops import (  # noqa: F401
    W4A16_ASYM, W4A16_SYM, W4A16_GROUP, W4A16_MAX_M, W4A16_MAX_TREE,
    W4A16_DEV_OK, W4A16_DEV_NONFINITE, W4A16_DEV_BAD_TREE, W4A16Error,
    W4A16_FAMILY_AUTO, W4A16_FAMILY_MMA_SYNC, W4A16_FAMILY_TCGEN05, W4A16_FAMILY_MMA_SYNC_S, W4A16_FAMILY_TCGEN05_OC,
    w4a16_pack, w4a16_unpack, w4a16_gemm, w4a16_gemm_workspace_bytes, w4a16_workspace_init,
    verify_accept, w4a16_status_string, w4a16_gemm_family, w4a16_silu_mul, w4a16_silu_mul_blocked,
    PackedLinear, pack_linear, alloc_workspace, w4a16_packed_bytes, Chain,
    w4a16_lmhead_argmax, w4a16_lmhead_workspace_bytes, alloc_lmhead_workspace,
    w4a16_tree_attention, w4a16_tree_attention_workspace_bytes, w4a16_kv_compact, w4a16_hadamard,
    PeerGroup, w4a16_peer_flag_bytes, w4a8_quantize_act, w4a8_workspace_bytes, w4a8_gemm,
)
