"""Same-name Python binding of the C ABI (include/w4a16.h) over torch tensors.

Each function checks dtypes/devices, passes raw device pointers and the current CUDA stream to
libw4a16.so, and raises W4A16Error on a non-zero status. Nothing here computes any part of the path.
"""
import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from ._lib import (  # noqa: F401
    lib, check, status_string, W4A16Error, W4A16_OK,
    W4A16_ASYM, W4A16_SYM, W4A16_GROUP, W4A16_MAX_M, W4A16_MAX_TREE,
    W4A16_DEV_OK, W4A16_DEV_NONFINITE, W4A16_DEV_BAD_TREE,
    W4A16_FAMILY_AUTO, W4A16_FAMILY_MMA_SYNC, W4A16_FAMILY_TCGEN05, W4A16_FAMILY_MMA_SYNC_S, W4A16_FAMILY_TCGEN05_OC,
    W4A16_OP_GEMM, W4A16_OP_SILU_MUL, W4A16_OP_ALLREDUCE, W4A16_OP_GEMM_SILU, W4A16_MAX_PEERS, W4A16Op, W4A16PeerGroup,
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


def _ptr_rows(t: torch.Tensor, name="tensor") -> int:
    """Pointer of a 2-D fp16 CUDA tensor whose rows are contiguous (a column slice of a wider buffer allowed)."""
    if not t.is_cuda:
        raise W4A16Error(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float16 or t.dim() != 2 or t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        raise W4A16Error(f"{name} must be a row-major fp16 [M, K] view")
    return t.data_ptr()


def _ldx(t: torch.Tensor) -> int:
    """Row stride of X for w4a16_op.ldx: 0 when contiguous."""
    return 0 if t.is_contiguous() or t.shape[0] == 1 else int(t.stride(0))


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
    """Y = X . W_hat through w4a16_gemm (family AUTO) or w4a16_gemm_ex (explicit family); an X whose rows are
    strided (a column slice of a wider buffer) goes through w4a16_gemm_strided and is read in place."""
    M, K = X.shape
    N = Y.shape[1]
    if Y.shape[0] != M:
        raise W4A16Error("Y must be [M, N]")
    ldx = _ldx(X)
    xp = _ptr_rows(X, "X") if ldx else _ptr(X, torch.float16, "X")
    args = (xp, _ptr(packed, None, "packed"), _ptr(Y, torch.float16, "Y"), M, K, N, group,
            mode, _ptr(workspace, None, "workspace"), workspace.numel() * workspace.element_size())
    if ldx:
        st = lib.w4a16_gemm_strided(args[0], ldx, *args[1:], family, _stream(stream))
    elif family == W4A16_FAMILY_AUTO:
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


def w4a16_lmhead_workspace_bytes(M: int, K: int, V: int) -> int:
    return int(lib.w4a16_lmhead_workspace_bytes(M, K, V))


def w4a16_lmhead_argmax(H, W_lm, out_argmax, workspace, out_max=None, stream=None):
    """out_argmax[m] (int32) = argmax_v H[m] . W_lm[v] (ties -> lowest id); out_max[m] (fp32) = that logit."""
    M, K = H.shape
    V = W_lm.shape[0]
    if W_lm.shape[1] != K or out_argmax.numel() < M:
        raise W4A16Error("w4a16_lmhead_argmax: shapes")
    check(lib.w4a16_lmhead_argmax(_ptr(H, torch.float16, "H"), _ptr(W_lm, torch.float16, "W_lm"), M, K, V,
                                  _ptr(out_argmax, torch.int32, "out_argmax"), _ptr(out_max, torch.float32, "out_max"),
                                  _ptr(workspace, None, "workspace"), workspace.numel() * workspace.element_size(),
                                  _stream(stream)), "w4a16_lmhead_argmax")


def alloc_lmhead_workspace(M_max: int, K: int, V: int, device=None) -> torch.Tensor:
    n = w4a16_lmhead_workspace_bytes(M_max, K, V)
    if n == 0:
        raise W4A16Error("w4a16_lmhead_workspace_bytes: bad shape")
    return torch.zeros(n, dtype=torch.uint8, device=device or "cuda")


def w4a16_tree_attention_workspace_bytes(M: int, L: int, Hq: int, Hkv: int, D: int = 128) -> int:
    return int(lib.w4a16_tree_attention_workspace_bytes(M, L, Hq, Hkv, D))


def w4a16_tree_attention(Q, Kc, Vc, parents, O, workspace, stream=None):
    """O [M, Hq, D] = tree-masked attention of Q [M, Hq, D] over Kc/Vc [L + M, Hkv, D]."""
    M, Hq, D = Q.shape
    Lt, Hkv, D2 = Kc.shape
    if D2 != D or tuple(Vc.shape) != tuple(Kc.shape) or tuple(O.shape) != tuple(Q.shape) or Lt < M:
        raise W4A16Error("w4a16_tree_attention: shapes")
    check(lib.w4a16_tree_attention(_ptr(Q, torch.float16, "Q"), _ptr(Kc, torch.float16, "Kc"), _ptr(Vc, torch.float16, "Vc"),
                                   _ptr(parents, torch.int32, "parents"), M, Lt - M, Hq, Hkv, D,
                                   _ptr(O, torch.float16, "O"), _ptr(workspace, None, "workspace"),
                                   workspace.numel() * workspace.element_size(), _stream(stream)), "w4a16_tree_attention")


def w4a16_kv_compact(Kc, Vc, L: int, accept_out, stream=None):
    """In place: cache rows L + k <- rows L + path[k-1] of the verify_accept result."""
    _, Hkv, D = Kc.shape
    check(lib.w4a16_kv_compact(_ptr(Kc, torch.float16, "Kc"), _ptr(Vc, torch.float16, "Vc"), L, Hkv, D,
                               _ptr(accept_out, torch.int32, "accept_out"), _stream(stream)), "w4a16_kv_compact")


def w4a16_hadamard(X, Y, block: int = 128, stream=None):
    """Y [M, K] = X rotated by the block Hadamard of size `block` along K. Y may be X."""
    M, K = X.shape
    check(lib.w4a16_hadamard(_ptr(X, torch.float16, "X"), _ptr(Y, torch.float16, "Y"), M, K, block, _stream(stream)),
          "w4a16_hadamard")


def w4a16_silu_mul(GU, out, stream=None):
    M, F2 = GU.shape
    check(lib.w4a16_silu_mul(_ptr(GU, torch.float16, "GU"), M, F2 // 2, _ptr(out, torch.float16, "out"),
                             _stream(stream)), "w4a16_silu_mul")


def w4a16_silu_mul_blocked(GU, out, block: int, stream=None):
    """out [M, F] = silu(gate) * up of GU [M, 2F] laid out in blocks of `block` gate then `block` up columns."""
    M, F2 = GU.shape
    check(lib.w4a16_silu_mul_blocked(_ptr(GU, torch.float16, "GU"), M, F2 // 2, int(block), _ptr(out, torch.float16, "out"),
                                     _stream(stream)), "w4a16_silu_mul_blocked")


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


class Chain:
    """A sequence of ops run as ONE persistent launch (include/w4a16.h: w4a16_chain_plan / w4a16_chain_run).

    ops: ("gemm", X [M,K] fp16, PackedLinear, Y [M,N] fp16), ("gemm_silu", X, PackedLinear, out [M,N/2] fp16)
    (gate-up with SiLU*mul fused; weight columns in [64 gate | 64 up] tiles) or ("silu_mul", GU [M,2F], out [M,F]).
    The plan (TMA descriptors, dependencies) is encoded once by the library into host memory and copied to
    the device here; the tensors must stay where they are while the chain is in use (references are kept)."""

    def __init__(self, ops, M: int, family=W4A16_FAMILY_AUTO, device=None, workspace=None, sms: Optional[int] = None):
        """workspace: optional zero-initialised uint8 tensor to use instead of a private one. Chains that run
        one after another on one stream may share it (each run re-arms its counters; partials are scratch).
        sms: tests only — plan for that many SMs and launch non-cooperatively, so that several chains can run
        side by side on one device (simulated tensor-parallel ranks)."""
        self.M, self.family, self.sms = M, family, sms
        self._keep = []
        arr = (W4A16Op * len(ops))()
        mode = W4A16_ASYM
        for i, op in enumerate(ops):
            if op[0] in ("gemm", "gemm_silu"):
                _, X, pl, Y = op
                ny = pl.N if op[0] == "gemm" else pl.N // 2
                if X.shape[0] != M or Y.shape[0] != M or X.shape[1] != pl.K or Y.shape[1] != ny:
                    raise W4A16Error(f"chain op {i}: shapes do not match M={M}, K={pl.K}, N={pl.N}")
                arr[i] = W4A16Op(W4A16_OP_GEMM if op[0] == "gemm" else W4A16_OP_GEMM_SILU, _ptr_rows(X, "X"),
                                 _ptr(pl.packed, None, "packed"), _ptr(Y, torch.float16, "Y"), pl.K, pl.N, pl.mode, _ldx(X))
                mode = pl.mode
                self._keep += [X, pl.packed, Y]
            elif op[0] == "allreduce":
                _, P, out, group = op
                if P.shape != out.shape or P.shape[0] != M:
                    raise W4A16Error(f"chain op {i}: allreduce shapes")
                N = P.shape[1]
                arr[i] = W4A16Op(W4A16_OP_ALLREDUCE, _ptr(P, torch.float16, "P"), ctypes.addressof(group.desc),
                                 _ptr(out, torch.float16, "out"), N, N, 0)
                self._keep += [P, out, group]
            elif op[0] == "silu_mul":
                _, GU, out = op
                F = out.shape[1]
                if GU.shape != (M, 2 * F) or out.shape[0] != M:
                    raise W4A16Error(f"chain op {i}: silu_mul shapes")
                arr[i] = W4A16Op(W4A16_OP_SILU_MUL, _ptr(GU, torch.float16, "GU"), None, _ptr(out, torch.float16, "out"),
                                 2 * F, F, 0)
                self._keep += [GU, out]
            else:
                raise W4A16Error(f"unknown chain op {op[0]!r}")
        self.n, self.mode = len(ops), mode
        nbytes = int(lib.w4a16_chain_plan_bytes(self.n))
        host = (ctypes.c_uint8 * nbytes)()
        if sms is None:
            check(lib.w4a16_chain_plan(ctypes.addressof(arr), self.n, M, family, ctypes.addressof(host), nbytes),
                  "w4a16_chain_plan")
        else:
            check(lib.w4a16_chain_plan_sms(ctypes.addressof(arr), self.n, M, family, ctypes.addressof(host), nbytes, sms),
                  "w4a16_chain_plan_sms")
        dev = torch.device(device) if device is not None else self._keep[0].device
        self.plan = torch.frombuffer(bytearray(host), dtype=torch.uint8).to(dev)
        wsb = int(lib.w4a16_chain_workspace_bytes(ctypes.addressof(arr), self.n, M, family) if sms is None else
                  lib.w4a16_chain_workspace_bytes_sms(ctypes.addressof(arr), self.n, M, family, sms))
        if wsb == 0:
            raise W4A16Error("w4a16_chain_workspace_bytes: bad chain")
        if workspace is not None:
            if workspace.numel() * workspace.element_size() < wsb:
                raise W4A16Error(f"chain workspace too small ({workspace.numel()} < {wsb} bytes)")
            self.ws = workspace
        else:
            self.ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)

    def __call__(self, stream=None):
        if self.sms is not None:
            check(lib.w4a16_chain_run_sms(self.plan.data_ptr(), self.n, self.M, self.mode, self.family,
                                          self.ws.data_ptr(), self.ws.numel(), self.sms, _stream(stream)),
                  "w4a16_chain_run_sms")
            return
        check(lib.w4a16_chain_run(self.plan.data_ptr(), self.n, self.M, self.mode, self.family, self.ws.data_ptr(),
                                  self.ws.numel(), _stream(stream)), "w4a16_chain_run")


def w4a16_peer_flag_bytes(flag_slots: int) -> int:
    return int(lib.w4a16_peer_flag_bytes(int(flag_slots)))


class _DevBuf:
    """A raw device allocation exposed to torch through __cuda_array_interface__ (uint8, 1-D)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                         "strides": None}


class PeerGroup:
    """A tensor-parallel group's symmetric regions (include/w4a16.h w4a16_peer_group), as seen by one rank.

    Each rank owns one device region of `nbytes`; the flag area of `flag_slots` ALLREDUCE ops sits at
    offset 0 and buffers are carved after it with alloc() — every rank must call alloc() with the same
    shapes in the same order, so each buffer has the same offset on every rank. Build with PeerGroup.ipc
    (one process per GPU, CUDA IPC) or PeerGroup.simulated (tests: `world` regions on one device)."""

    def __init__(self, bases, local: torch.Tensor, nbytes: int, flag_slots: int, world: int, rank: int, closer=None,
                 mc_base: Optional[int] = None):
        if not 1 <= world <= W4A16_MAX_PEERS or not 0 <= rank < world or len(bases) != world:
            raise W4A16Error(f"peer group: world={world}, rank={rank}")
        self.world, self.rank, self.nbytes, self.flag_slots = world, rank, nbytes, flag_slots
        self.local = local
        self.desc = W4A16PeerGroup()
        for q, b in enumerate(bases):
            self.desc.base[q] = b
        self.desc.bytes, self.desc.flag_offset, self.desc.flag_slots = nbytes, 0, flag_slots
        self.desc.world, self.desc.rank = world, rank
        self.desc.mc_base = mc_base
        self.kind = "nvls" if mc_base else "peer"
        self._next = (w4a16_peer_flag_bytes(flag_slots) + 255) // 256 * 256
        self._closer = closer

    def alloc(self, *shape, dtype=torch.float16) -> torch.Tensor:
        """The next symmetric buffer (same offset on every rank), 256-byte aligned."""
        n = 1
        for d in shape:
            n *= d
        nb = n * torch.empty((), dtype=dtype).element_size()
        if self._next + nb > self.nbytes:
            raise W4A16Error(f"peer region full ({self._next} + {nb} > {self.nbytes} bytes)")
        t = self.local[self._next: self._next + nb].view(dtype).view(*shape)
        self._next += (nb + 255) // 256 * 256
        return t

    def peer_region(self, q: int) -> torch.Tensor:
        """Rank q's whole region as mapped in this process (uint8 view; tests and diagnostics)."""
        if q == self.rank:
            return self.local
        return torch.as_tensor(_DevBuf(self.desc.base[q], self.nbytes), device=self.local.device)

    @staticmethod
    def simulated(world: int, nbytes: int, flag_slots: int, device=None):
        """Tests: `world` zero-filled regions on ONE device, one PeerGroup per simulated rank."""
        regs = [torch.zeros(nbytes, dtype=torch.uint8, device=device) for _ in range(world)]
        bases = [r.data_ptr() for r in regs]
        groups = [PeerGroup(bases, regs[r], nbytes, flag_slots, world, r) for r in range(world)]
        for g in groups:
            g._regions = regs   # keep every region alive
        return groups

    @staticmethod
    def ipc(nbytes: int, flag_slots: int, group=None):
        """One process per GPU: allocate this rank's region, exchange CUDA IPC handles over `group` (any
        torch.distributed backend) and map every peer's region."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * 64)()
        st = lib.w4a16_ipc_alloc(nbytes, ctypes.byref(ptr), handle)
        # every step is agreed on by all ranks (a rank that fails still takes part in the collectives, so
        # no rank is left waiting in one)
        handles = [None] * world
        dist.all_gather_object(handles, (st, bytes(handle)), group=group)
        bases, opened = [], []

        def closer():
            for p in opened:
                lib.w4a16_ipc_close(p)
            if st == W4A16_OK:
                lib.w4a16_ipc_free(ptr.value)
        if any(s != W4A16_OK for s, _ in handles):
            closer()
            raise W4A16Error(f"w4a16_ipc_alloc failed on rank(s) {[q for q, (s, _) in enumerate(handles) if s != W4A16_OK]}")
        err = W4A16_OK
        for q, (_, h) in enumerate(handles):
            if q == rank:
                bases.append(ptr.value)
                continue
            hb = (ctypes.c_uint8 * 64).from_buffer_copy(h)
            p = ctypes.c_void_p()
            e = lib.w4a16_ipc_open(hb, ctypes.byref(p))
            if e != W4A16_OK:
                err = e
                bases.append(None)
                continue
            bases.append(p.value)
            opened.append(p.value)
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        if any(e != W4A16_OK for e in errs):
            closer()
            raise W4A16Error(f"w4a16_ipc_open failed on rank(s) {[q for q, e in enumerate(errs) if e != W4A16_OK]}")
        local = torch.as_tensor(_DevBuf(ptr.value, nbytes), device=torch.device("cuda", torch.cuda.current_device()))
        return PeerGroup(bases, local, nbytes, flag_slots, world, rank, closer)

    @staticmethod
    def mc_supported() -> bool:
        return bool(lib.w4a16_mc_supported())

    @staticmethod
    def mc(nbytes: int, flag_slots: int, group=None):
        """One process per GPU, NVLS: rank 0 creates a multicast object for the group (fabric handle sent over
        `group`, any torch.distributed backend), every rank adds its device, then binds its own region to it
        and maps the multicast range (include/w4a16.h w4a16_mc_*). The ALLREDUCE ops then bump tile counters
        with one multimem.red and reduce with multimem.ld_reduce; peers' regions are never mapped."""
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0

        def agree(ok: bool, what: str):
            flags = [ok]
            if world > 1:
                flags = [None] * world
                dist.all_gather_object(flags, ok, group=group)
            if not all(flags):
                raise W4A16Error(f"{what} failed on rank(s) {[q for q, f in enumerate(flags) if not f]}")
        agree(bool(lib.w4a16_mc_supported()), "w4a16_mc_supported")
        mc = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * 64)()
        st = lib.w4a16_mc_create(nbytes, world, handle, ctypes.byref(mc)) if rank == 0 else W4A16_OK
        hs = [(st, bytes(handle))]
        if world > 1:
            hs = [None] * world
            dist.all_gather_object(hs, (st, bytes(handle)), group=group)
        agree(hs[0][0] == W4A16_OK, "w4a16_mc_create (rank 0)")
        if rank != 0:
            hb = (ctypes.c_uint8 * 64).from_buffer_copy(hs[0][1])
            st = lib.w4a16_mc_import(hb, nbytes, world, ctypes.byref(mc))
            agree(st == W4A16_OK, "w4a16_mc_import")
        st = lib.w4a16_mc_add_device(mc)
        agree(st == W4A16_OK, "w4a16_mc_add_device")   # every device added before any rank binds
        uc, mva = ctypes.c_void_p(), ctypes.c_void_p()
        st = lib.w4a16_mc_bind(mc, nbytes, ctypes.byref(uc), ctypes.byref(mva))
        agree(st == W4A16_OK, "w4a16_mc_bind")
        if world > 1:
            dist.barrier(group=group)   # every rank bound before the first multicast access

        def closer():
            lib.w4a16_mc_free(mc, uc, mva, nbytes)
        local = torch.as_tensor(_DevBuf(uc.value, nbytes), device=torch.device("cuda", torch.cuda.current_device()))
        bases = [uc.value if q == rank else None for q in range(world)]
        return PeerGroup(bases, local, nbytes, flag_slots, world, rank, closer, mc_base=mva.value)

    def close(self):
        if self._closer is not None:
            self._closer()
            self._closer = None


# ---- W4A8 (include/w4a16.h) ----
def w4a8_quantize_act(X, Xq, sx, xsum, stream=None):
    """Per-token int8 activations: X fp16 [M, K] -> Xq int8 [M, K], sx fp32 [M], xsum int32 [M, K/128]."""
    M, K = X.shape
    if Xq.dtype != torch.int8 or sx.dtype != torch.float32 or xsum.dtype != torch.int32:
        raise W4A16Error("w4a8_quantize_act: dtypes")
    if tuple(Xq.shape) != (M, K) or sx.numel() < M or tuple(xsum.shape) != (M, K // 128):
        raise W4A16Error("w4a8_quantize_act: shapes")
    check(lib.w4a8_quantize_act(_ptr(X, torch.float16, "X"), M, K, Xq.data_ptr(), sx.data_ptr(), xsum.data_ptr(),
                                _stream(stream)), "w4a8_quantize_act")


def w4a8_workspace_bytes(M: int, K: int, N: int) -> int:
    return int(lib.w4a8_workspace_bytes(M, K, N))


def w4a8_gemm(Xq, sx, xsum, packed, Y, workspace, stream=None, impl: int = 0):
    """Y [M, N] fp16 = W4A8 GEMM of the quantised activations with a SYM w4a16_pack blob (K x N).
    impl (tests / A-B only, the w4a8_gemm_ex hook): 0 = auto, 1 = family-A pipeline (M <= 16), 2 = round-1 kernel."""
    M, K = Xq.shape
    N = Y.shape[1]
    if Xq.dtype != torch.int8 or Y.shape[0] != M:
        raise W4A16Error("w4a8_gemm: shapes / dtypes")
    args = (Xq.data_ptr(), sx.data_ptr(), xsum.data_ptr(), _ptr(packed, None, "packed"), _ptr(Y, torch.float16, "Y"), M, K, N,
            workspace.data_ptr(), workspace.numel() * workspace.element_size())
    if impl == 0:
        check(lib.w4a8_gemm(*args, _stream(stream)), "w4a8_gemm")
    else:
        check(lib.w4a8_gemm_ex(*args, int(impl), _stream(stream)), "w4a8_gemm_ex")
