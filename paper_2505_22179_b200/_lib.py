"""ctypes binding of libw4a16.so — the C ABI declared in include/w4a16.h.

Argument marshalling only: every step of the path runs in the sm_100a kernels behind the ABI. There is
no CPU fallback: if the shared library is missing the import of this module raises.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# W4A16_LIB=<name> loads libw4a16_<name>.so (diagnostic builds only: make diag); never set by tests or bench
LIB_PATH = os.path.join(_HERE, f"libw4a16_{os.environ['W4A16_LIB']}.so" if os.environ.get("W4A16_LIB") else "libw4a16.so")

W4A16_OK = 0
W4A16_ASYM = 0
W4A16_SYM = 1
W4A16_DEV_OK = 0
W4A16_DEV_NONFINITE = 1
W4A16_DEV_BAD_TREE = 2
W4A16_GROUP = 128
W4A16_MAX_M = 64
W4A16_MAX_TREE = 1024
W4A16_MAX_N = 1048576
W4A16_AR_MAX_TILES = 128
W4A16_FAMILY_AUTO, W4A16_FAMILY_MMA_SYNC, W4A16_FAMILY_TCGEN05, W4A16_FAMILY_MMA_SYNC_S, W4A16_FAMILY_TCGEN05_OC = -1, 0, 1, 2, 3

# Every symbol include/w4a16.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = (
    "w4a16_packed_bytes",
    "w4a16_pack",
    "w4a16_unpack",
    "w4a16_gemm_workspace_bytes",
    "w4a16_workspace_init",
    "w4a16_gemm",
    "w4a16_gemm_ex",
    "w4a16_gemm_strided",
    "verify_accept",
    "w4a16_status_string",
    "w4a16_gemm_family",
    "w4a16_silu_mul",
    "w4a16_silu_mul_blocked",
    "w4a16_chain_plan_bytes",
    "w4a16_chain_workspace_bytes",
    "w4a16_chain_plan",
    "w4a16_chain_run",
    "w4a16_lmhead_workspace_bytes",
    "w4a16_lmhead_argmax",
    "w4a16_tree_attention_workspace_bytes",
    "w4a16_tree_attention",
    "w4a16_kv_compact",
    "w4a16_hadamard",
    "w4a16_peer_flag_bytes",
    "w4a16_ipc_alloc",
    "w4a16_ipc_open",
    "w4a16_ipc_close",
    "w4a16_ipc_free",
    "w4a16_mc_supported",
    "w4a16_mc_create",
    "w4a16_mc_import",
    "w4a16_mc_add_device",
    "w4a16_mc_bind",
    "w4a16_mc_free",
    "w4a8_quantize_act",
    "w4a8_workspace_bytes",
    "w4a8_gemm",
)
W4A16_OP_GEMM, W4A16_OP_SILU_MUL, W4A16_OP_ALLREDUCE, W4A16_OP_GEMM_SILU = 0, 1, 2, 3
W4A16_MAX_PEERS = 8


class W4A16Op(ctypes.Structure):
    """struct w4a16_op of include/w4a16.h."""
    _fields_ = [("kind", ctypes.c_int), ("X", ctypes.c_void_p), ("packed", ctypes.c_void_p), ("Y", ctypes.c_void_p),
                ("K", ctypes.c_int), ("N", ctypes.c_int), ("mode", ctypes.c_int), ("ldx", ctypes.c_int)]


class W4A16PeerGroup(ctypes.Structure):
    """struct w4a16_peer_group of include/w4a16.h (host side; read by w4a16_chain_plan only)."""
    _fields_ = [("base", ctypes.c_void_p * W4A16_MAX_PEERS), ("bytes", ctypes.c_size_t), ("flag_offset", ctypes.c_size_t),
                ("flag_slots", ctypes.c_int), ("world", ctypes.c_int), ("rank", ctypes.c_int), ("mc_base", ctypes.c_void_p)]


class W4A16Error(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built: run `make` (or __graft_entry__.build()). "
            "The W4A16 path has no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    lib.w4a16_packed_bytes.argtypes = [i32, i32, i32, i32]
    lib.w4a16_packed_bytes.restype = sz
    lib.w4a16_pack.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp]
    lib.w4a16_unpack.argtypes = [vp, i32, i32, i32, i32, vp, vp]
    lib.w4a16_gemm_workspace_bytes.argtypes = [i32, i32, i32, i32]
    lib.w4a16_gemm_workspace_bytes.restype = sz
    lib.w4a16_workspace_init.argtypes = [vp, sz, vp]
    lib.w4a16_gemm.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp, sz, vp]
    lib.w4a16_gemm_ex.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp, sz, i32, vp]
    if hasattr(lib, "w4a16_gemm_strided"):
        lib.w4a16_gemm_strided.argtypes = [vp, i32, vp, vp, i32, i32, i32, i32, i32, vp, sz, i32, vp]
        lib.w4a16_gemm_strided.restype = i32
    lib.verify_accept.argtypes = [vp, vp, vp, i32, vp, vp]
    lib.w4a16_status_string.argtypes = [i32]
    lib.w4a16_status_string.restype = ctypes.c_char_p
    lib.w4a16_gemm_family.argtypes = [i32, i32, i32]
    lib.w4a16_silu_mul.argtypes = [vp, i32, i32, vp, vp]
    lib.w4a16_silu_mul_blocked.argtypes = [vp, i32, i32, i32, vp, vp]
    lib.w4a16_lmhead_workspace_bytes.argtypes = [i32, i32, i32]
    lib.w4a16_lmhead_workspace_bytes.restype = sz
    lib.w4a16_lmhead_argmax.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp, sz, vp]
    lib.w4a16_lmhead_argmax.restype = i32
    lib.w4a16_tree_attention_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
    lib.w4a16_tree_attention_workspace_bytes.restype = sz
    lib.w4a16_tree_attention.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, vp, vp, sz, vp]
    lib.w4a16_tree_attention.restype = i32
    lib.w4a16_kv_compact.argtypes = [vp, vp, i32, i32, i32, vp, vp]
    lib.w4a16_kv_compact.restype = i32
    lib.w4a16_hadamard.argtypes = [vp, vp, i32, i32, i32, vp]
    lib.w4a16_hadamard.restype = i32
    lib.w4a8_quantize_act.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    lib.w4a8_quantize_act.restype = i32
    lib.w4a8_workspace_bytes.argtypes = [i32, i32, i32]
    lib.w4a8_workspace_bytes.restype = sz
    lib.w4a8_gemm.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, vp, sz, vp]
    lib.w4a8_gemm.restype = i32
    lib.w4a16_chain_plan_bytes.argtypes = [i32]
    lib.w4a16_chain_plan_bytes.restype = sz
    lib.w4a16_chain_workspace_bytes.argtypes = [vp, i32, i32, i32]
    lib.w4a16_chain_workspace_bytes.restype = sz
    lib.w4a16_chain_plan.argtypes = [vp, i32, i32, i32, vp, sz]
    lib.w4a16_chain_run.argtypes = [vp, i32, i32, i32, i32, vp, sz, vp]
    if not hasattr(lib, "w4a16_chain_run_sms") and os.environ.get("W4A16_LIB"):
        return lib   # an older diagnostics build (A/B timing only): chains without ALLREDUCE ops
    lib.w4a16_peer_flag_bytes.argtypes = [i32]
    lib.w4a16_peer_flag_bytes.restype = sz
    lib.w4a16_ipc_alloc.argtypes = [sz, ctypes.POINTER(vp), vp]
    lib.w4a16_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
    lib.w4a16_ipc_close.argtypes = [vp]
    lib.w4a16_ipc_free.argtypes = [vp]
    if not hasattr(lib, "w4a16_mc_supported") and os.environ.get("W4A16_LIB"):
        return lib   # an older A/B build without the NVLS functions
    lib.w4a16_mc_supported.argtypes = []
    lib.w4a16_mc_create.argtypes = [sz, i32, vp, ctypes.POINTER(vp)]
    lib.w4a16_mc_import.argtypes = [vp, sz, i32, ctypes.POINTER(vp)]
    lib.w4a16_mc_add_device.argtypes = [vp]
    lib.w4a16_mc_bind.argtypes = [vp, sz, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    lib.w4a16_mc_free.argtypes = [vp, vp, vp, sz]
    # test hooks (exported, not in the header): chains planned / run for a given SM count, non-cooperatively
    lib.w4a16_chain_workspace_bytes_sms.argtypes = [vp, i32, i32, i32, i32]
    lib.w4a16_chain_workspace_bytes_sms.restype = sz
    lib.w4a16_chain_plan_sms.argtypes = [vp, i32, i32, i32, vp, sz, i32]
    lib.w4a16_chain_check_sms.argtypes = [vp, i32, i32, i32, i32]
    lib.w4a16_chain_check_sms.restype = i32
    lib.w4a8_gemm_ex.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, vp, sz, i32, vp]
    lib.w4a8_gemm_ex.restype = i32
    lib.w4a16_chain_run_sms.argtypes = [vp, i32, i32, i32, i32, vp, sz, i32, vp]
    for name in ("w4a16_ipc_alloc", "w4a16_ipc_open", "w4a16_ipc_close", "w4a16_ipc_free", "w4a16_mc_supported",
                 "w4a16_mc_create", "w4a16_mc_import", "w4a16_mc_add_device", "w4a16_mc_bind", "w4a16_mc_free", "w4a16_chain_plan_sms",
                 "w4a16_chain_run_sms", "w4a16_chain_plan", "w4a16_chain_run", "w4a16_pack", "w4a16_unpack", "w4a16_workspace_init", "w4a16_gemm", "w4a16_gemm_ex", "verify_accept",
                 "w4a16_gemm_family", "w4a16_silu_mul", "w4a16_silu_mul_blocked"):
        getattr(lib, name).restype = i32
    return lib


lib = _load()


def status_string(status: int) -> str:
    return lib.w4a16_status_string(int(status)).decode()


def check(status: int, what: str) -> None:
    if status != W4A16_OK:
        raise W4A16Error(f"{what}: {status_string(status)} ({status})")
