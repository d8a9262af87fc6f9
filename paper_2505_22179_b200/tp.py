"""Tensor-parallel W4A16 verify stack (BASELINE.json configs 4-5).

One process per GPU. Megatron-style partition of each Llama decoder layer's linear layers:
  * column-parallel (split N, no communication): QKV (head-aligned: rank r owns q heads
    [r*nq/t, (r+1)*nq/t) and kv heads [r*nkv/t, ...)), gate-up (rank r owns the matching gate AND up
    columns, given by make_weight as [gate_r | up_r] and stored interleaved in [64 gate | 64 up] tiles so the
    gate-up GEMM's epilogue can apply SiLU*mul);
  * row-parallel (split K): O (rank's heads) and down (rank's FFN slice); each rank produces a partial
    Y[M, hidden] that an all-reduce (NCCL over NVLink/NVSwitch, via torch.distributed) sums.
Data flow of one verify forward (the dependencies of a real decoder stack: the target
verifies the draft "in one forward pass"):
  h_0 = x_in;  per layer l:  qkv = h_l . W_qkv;  o = qkv[:, :K_o] . W_o  (the attention stub: the rank's query
  columns stand in for the attention output, whose kernel is SURVEY §8(f) f2 and outside the timed stack);
  [all-reduce];  act = silu(gate) * up of gu = o . W_gu (fused into the gate-up GEMM's epilogue in chains:
  the gate-up weight is stored in 128-column tiles of [64 gate | 64 up]);  h_{l+1} = act . W_down  [all-reduce].
Attention, norms and residual adds are outside the hot path. So every GEMM reads what the previous one
wrote: QKV -> O -> gate-up -> SiLU*mul -> down -> QKV of the next layer (read-after-write edges, which a
persistent chain must honour). Because the norms are absent, `calibrate=True` rescales each synthetic weight
once at build time by a power of two so that its output has RMS in [1/sqrt(2), sqrt(2)] on the actual data flow (a stand-in for RMSNorm that keeps
activations O(1) through 80 layers). Every compute step is a libw4a16.so kernel; torch supplies memory,
streams, CUDA graphs and the process group.
"""
import math
from dataclasses import dataclass
from typing import Callable, List, Optional

import torch
import torch.distributed as dist

from .ops import (W4A16_ASYM, Chain, PackedLinear, PeerGroup, W4A16Error, alloc_workspace, pack_linear,
                  verify_accept, w4a16_peer_flag_bytes, w4a16_silu_mul_blocked)

SILU_BLOCK = 64   # gate-up weight columns are stored in 128-column tiles of [64 gate | 64 up] (W4A16_OP_GEMM_SILU)


def interleave_gate_up(W: torch.Tensor) -> torch.Tensor:
    """[K, 2F] in the logical [gate | up] column order -> [64 gate | 64 up] blocks (the stored layout)."""
    K, F2 = W.shape
    F = F2 // 2
    return W.view(K, 2, F // SILU_BLOCK, SILU_BLOCK).permute(0, 2, 1, 3).reshape(K, F2)


@dataclass(frozen=True)
class ModelDims:
    name: str
    hidden: int
    ffn: int
    n_q: int
    n_kv: int
    head: int
    layers: int

    @property
    def qkv_out(self):
        return (self.n_q + 2 * self.n_kv) * self.head


LLAMA3_8B = ModelDims("llama3-8b", 4096, 14336, 32, 8, 128, 32)
LLAMA3_70B = ModelDims("llama3-70b", 8192, 28672, 64, 8, 128, 80)
MATRICES = ("qkv", "o", "gate_up", "down")


def _split(total: int, t: int, r: int, align: int = 128):
    if total % t or (total // t) % align:
        raise ValueError(f"{total} does not split into {t} shards aligned to {align}")
    s = total // t
    return r * s, (r + 1) * s


def shard_plan(d: ModelDims, t: int, r: int) -> dict:
    """Per-rank GEMM shapes (K, N) and the column/row ranges of the full matrices they cover.

    'cols' lists (start, stop) column ranges of the full [K, N] weight, concatenated in order;
    'rows' is the (start, stop) row (K) range. All ranges are multiples of 128."""
    if d.n_kv % t or d.n_q % t:
        raise ValueError(f"tp={t} must divide the head counts")
    hq, hk = d.n_q // t, d.n_kv // t
    q = (r * hq * d.head, (r + 1) * hq * d.head)
    k0 = d.n_q * d.head
    kk = (k0 + r * hk * d.head, k0 + (r + 1) * hk * d.head)
    v0 = k0 + d.n_kv * d.head
    vv = (v0 + r * hk * d.head, v0 + (r + 1) * hk * d.head)
    g = _split(d.ffn, t, r)
    u = (d.ffn + g[0], d.ffn + g[1])
    o_rows = _split(d.n_q * d.head, t, r)
    return {
        "qkv": {"K": d.hidden, "N": (hq + 2 * hk) * d.head, "rows": (0, d.hidden), "cols": [q, kk, vv],
                "full": (d.hidden, d.qkv_out)},
        "o": {"K": d.n_q * d.head // t, "N": d.hidden, "rows": o_rows, "cols": [(0, d.hidden)],
              "full": (d.n_q * d.head, d.hidden)},
        "gate_up": {"K": d.hidden, "N": 2 * d.ffn // t, "rows": (0, d.hidden), "cols": [g, u],
                    "full": (d.hidden, 2 * d.ffn)},
        "down": {"K": d.ffn // t, "N": d.hidden, "rows": g, "cols": [(0, d.hidden)], "full": (d.ffn, d.hidden)},
    }


def shard_of(W_full: torch.Tensor, spec: dict) -> torch.Tensor:
    """The rank-local [K_r, N_r] weight of a full [K, N] weight under shard_plan (any device)."""
    r0, r1 = spec["rows"]
    return torch.cat([W_full[r0:r1, c0:c1] for c0, c1 in spec["cols"]], dim=1).contiguous()


def weight_bytes(d: ModelDims, t: int, n_layers: Optional[int] = None, sym: bool = False) -> int:
    """Algorithmic weight bytes streamed by ONE rank per verify forward (codes + scales (+ zeros))."""
    plan = shard_plan(d, t, 0)
    per = sum(s["K"] * s["N"] // 2 + (s["K"] // 128) * s["N"] * (2 if sym else 4) for s in plan.values())
    return per * (n_layers if n_layers is not None else d.layers)


class VerifyStack:
    """The rank-local shard of an n_layers-deep W4A16 verify stack, resident in HBM.

    make_weight(layer, name, K, N, out) fills `out` (fp16 [K, N] CUDA tensor) with the rank-local weight;
    it is packed with w4a16_pack and dropped, so only the int4 shards stay resident."""

    def __init__(self, dims: ModelDims, n_layers: int, M_max: int, make_weight: Callable, tp_size: int = 1,
                 tp_rank: int = 0, group=None, mode: int = W4A16_ASYM, device=None, allreduce: str = "nccl",
                 peer_group: Optional[PeerGroup] = None, chain_sms: Optional[int] = None,
                 calibrate: Optional[torch.Tensor] = None):
        """allreduce: "nccl" or "fused" (tp > 1). peer_group / chain_sms: tests only — a PeerGroup.simulated
        rank and the SM share of its chains, to run several ranks side by side on one GPU.
        calibrate: optional [Mc, hidden] fp16 input; each weight is scaled once (before packing) so that its
        GEMM output on the forward's data flow from that input has unit RMS (module docstring)."""
        if allreduce not in ("nccl", "fused"):
            raise ValueError(f"allreduce={allreduce!r}")
        self.d, self.n_layers, self.M_max = dims, n_layers, M_max
        self.t, self.r, self.group, self.mode = tp_size, tp_rank, group, mode
        self.fused = allreduce == "fused" and tp_size > 1
        self.chain_sms = chain_sms
        self.device = torch.device(device or "cuda")
        self.plan = shard_plan(dims, tp_size, tp_rank)
        biggest = max(s["K"] * s["N"] for s in self.plan.values())
        tmp = torch.empty(biggest, dtype=torch.float16, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.layers: List[dict] = []
        self.calib_scale: List[dict] = []
        cal = None if calibrate is None else _Calibration(self, calibrate)
        for l in range(n_layers):
            mats = {}
            for name in MATRICES:
                s = self.plan[name]
                W = tmp[: s["K"] * s["N"]].view(s["K"], s["N"])
                make_weight(l, name, s["K"], s["N"], W)   # logical column order ([gate | up] for gate-up)
                if name == "gate_up":
                    W.copy_(interleave_gate_up(W))
                mats[name] = pack_linear(W, mode=mode, dev_status=self.status)
                if cal is not None:
                    mats[name] = cal.step(l, name, W, mats[name])
            self.layers.append(mats)
        del tmp, cal
        torch.cuda.synchronize(self.device)
        f16 = dict(dtype=torch.float16, device=self.device)
        P = self.plan
        # the forward's input hidden state (caller fills) and per-layer scratch outputs (module docstring)
        self.x_in = torch.zeros(M_max, P["qkv"]["K"], **f16)
        self.y_qkv = torch.zeros(M_max, P["qkv"]["N"], **f16)
        self.y_gu = torch.empty(M_max, P["gate_up"]["N"], **f16)
        self.act = torch.empty(M_max, P["down"]["K"], **f16)
        if self.fused:
            # row-parallel partials live in the symmetric region (same offsets on every rank); the reduced
            # outputs are ordinary local buffers
            slots = 2 * n_layers
            nbytes = w4a16_peer_flag_bytes(slots) + 2 * M_max * (P["o"]["N"] + P["down"]["N"]) + 4096
            self.peers = peer_group if peer_group is not None else _peer_group(nbytes, slots, group)
            self.y_o = self.peers.alloc(M_max, P["o"]["N"])
            self.y_down = self.peers.alloc(M_max, P["down"]["N"])
            self.y_o_red = torch.empty(M_max, P["o"]["N"], **f16)
            self.y_down_red = torch.empty(M_max, P["down"]["N"], **f16)
        else:
            self.peers = None
            self.y_o = torch.zeros(M_max, P["o"]["N"], **f16)
            self.y_down = torch.zeros(M_max, P["down"]["N"], **f16)
            self.y_o_red, self.y_down_red = self.y_o, self.y_down   # NCCL reduces in place
        i32 = dict(dtype=torch.int32, device=self.device)
        self.tokens = torch.zeros(M_max, **i32)
        self.parents = torch.full((M_max,), -1, **i32)
        self.parents[1:] = torch.arange(M_max - 1, device=self.device, dtype=torch.int32)
        self.argmax = torch.zeros(M_max, **i32)
        self.accept_out = torch.zeros(3 + M_max, **i32)
        self.ws = alloc_workspace(M_max, [(s["K"], s["N"]) for s in P.values()], device=self.device)
        self.graphs = {}
        self.capturable = True
        self.use_chains = True
        self._chains = {}

    @property
    def weight_bytes(self) -> int:
        return sum(pl.weight_bytes for L in self.layers for pl in L.values())

    def _allreduce(self, y: torch.Tensor):
        if self.t > 1:
            dist.all_reduce(y, group=self.group)

    def layer_input(self, l: int, M: int) -> torch.Tensor:
        """h_l: the QKV input of layer l (x_in for layer 0, else the previous layer's reduced down output)."""
        return self.x_in[:M] if l == 0 else self.y_down_red[:M]

    def q_part(self, M: int) -> torch.Tensor:
        """The attention stub: the rank's query columns of the QKV output (a strided [M, K_o] view)."""
        return self.y_qkv[:M, : self.plan["o"]["K"]]

    def _layer_ops(self, L, M, l=0):
        """The layer's ops between its all-reduces: [QKV, O] and [gate-up, SiLU*mul, down]; with the fused
        all-reduce each segment ends with its ALLREDUCE op (partial in the peer region -> reduced output)."""
        a = [("gemm", self.layer_input(l, M), L["qkv"], self.y_qkv[:M]), ("gemm", self.q_part(M), L["o"], self.y_o[:M])]
        b = [("gemm_silu", self.y_o_red[:M], L["gate_up"], self.act[:M]),   # gate-up with SiLU*mul fused
             ("gemm", self.act[:M], L["down"], self.y_down[:M])]
        if self.fused:
            a.append(("allreduce", self.y_o[:M], self.y_o_red[:M], self.peers))
            b.append(("allreduce", self.y_down[:M], self.y_down_red[:M], self.peers))
        return a, b

    def chains(self, M: int):
        """Persistent chains for width M (include/w4a16.h w4a16_chain_*): the whole stack in ONE launch at
        tp = 1; at tp > 1 one launch per segment between all-reduces (mma.sync families, M <= 16). None for
        M > 16 or where a shard is too small to give every CTA a unit: then every op is launched on its own."""
        if M not in self._chains:
            if M > 16:   # chains serve the mma.sync families; the tcgen05 family is launched op by op
                self._chains[M] = None
                return None
            try:
                segs = [self._layer_ops(L, M, l) for l, L in enumerate(self.layers)]
                if self.t == 1 or self.fused:   # the whole forward in one launch
                    self._chains[M] = [Chain([op for a, b in segs for op in a + b], M, device=self.device,
                                             sms=self.chain_sms)]
                else:
                    # the per-segment chains run one after another on one stream: they share one workspace
                    first = [Chain(seg, M, device=self.device) for seg in segs[0]]
                    ws = max((c.ws for c in first), key=lambda t: t.numel())
                    self._chains[M] = [Chain(seg, M, device=self.device, workspace=ws) for a, b in segs
                                       for seg in (a, b)]
            except W4A16Error:
                self._chains[M] = None
        return self._chains[M]

    def forward(self, M: int, stream=None):
        """One verify forward at width M (M = draft nodes + root), then greedy acceptance. Async."""
        if not 1 <= M <= self.M_max:
            raise ValueError(f"M={M} outside [1, {self.M_max}]")
        ch = self.chains(M) if self.use_chains else None
        if ch is not None:
            if self.t == 1 or self.fused:
                ch[0](stream)
            else:
                for i, c in enumerate(ch):
                    c(stream)
                    self._allreduce(self.y_o[:M] if i % 2 == 0 else self.y_down[:M])
            verify_accept(self.tokens[:M], self.parents[:M], self.argmax[:M], self.accept_out[:3 + M], stream)
            return
        ws = self.ws
        # op by op (M > 16, or chains off): NCCL all-reduces; with the fused layout the partial is first
        # copied to the reduced buffer (the ALLREDUCE op exists only inside chains)
        o_out, d_out = (self.y_o_red[:M], self.y_down_red[:M]) if self.fused else (self.y_o[:M], self.y_down[:M])
        for l, L in enumerate(self.layers):
            L["qkv"](self.layer_input(l, M), self.y_qkv[:M], ws, stream)
            L["o"](self.q_part(M), self.y_o[:M], ws, stream)   # the strided query view, read in place
            if self.fused:
                o_out.copy_(self.y_o[:M])
            self._allreduce(o_out)
            L["gate_up"](o_out, self.y_gu[:M], ws, stream)
            w4a16_silu_mul_blocked(self.y_gu[:M], self.act[:M], SILU_BLOCK, stream)
            L["down"](self.act[:M], self.y_down[:M], ws, stream)
            if self.fused:
                d_out.copy_(self.y_down[:M])
            self._allreduce(d_out)
        verify_accept(self.tokens[:M], self.parents[:M], self.argmax[:M], self.accept_out[:3 + M], stream)

    def launches_per_forward(self, M: int = None) -> int:
        """libw4a16 kernel launches per forward: one chain (tp = 1, or the fused all-reduce) or two per layer
        (tp > 1 with NCCL) plus the acceptance; without chains 4 GEMMs + SiLU*mul per layer plus the acceptance."""
        if M is not None and self.use_chains and self.chains(M) is not None:
            return len(self.chains(M)) + 1
        return 5 * self.n_layers + 1

    def capture(self, M: int) -> torch.cuda.CUDAGraph:
        """Capture forward(M) as a CUDA graph (after one eager warm-up on the capture stream). With
        capturable = False (a process group whose all-reduce cannot be captured, e.g. gloo in the tests of
        bench.py's multi-rank path) an object whose replay() runs forward(M) eagerly is returned instead."""
        if M in self.graphs:
            return self.graphs[M]
        if not self.capturable:
            self.graphs[M] = _Eager(self, M)
            return self.graphs[M]
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.forward(M)
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.forward(M)
        torch.cuda.synchronize(self.device)
        self.graphs[M] = g
        return g

    def set_tree(self, tokens, parents, argmax):
        n = len(tokens)
        self.tokens[:n].copy_(torch.as_tensor(tokens, dtype=torch.int32))
        self.parents[:n].copy_(torch.as_tensor(parents, dtype=torch.int32))
        self.argmax[:n].copy_(torch.as_tensor(argmax, dtype=torch.int32))

    def verify_host(self, M: int, host_in: dict, host_out: dict, graph: Optional[torch.cuda.CUDAGraph] = None):
        """End-to-end step through the public API: pinned host inputs -> device, forward (graph replay if
        given), accepted length / path / last hidden state -> pinned host. Async on the current stream."""
        self.x_in[:M].copy_(host_in["x_in"][:M], non_blocking=True)
        self.tokens[:M].copy_(host_in["tokens"][:M], non_blocking=True)
        self.parents[:M].copy_(host_in["parents"][:M], non_blocking=True)
        self.argmax[:M].copy_(host_in["argmax"][:M], non_blocking=True)
        if graph is not None:
            graph.replay()
        else:
            self.forward(M)
        host_out["accept"][:3 + M].copy_(self.accept_out[:3 + M], non_blocking=True)
        host_out["y"][:M].copy_(self.y_down_red[:M], non_blocking=True)

    def h2d_bytes(self, M: int) -> int:
        return 2 * M * self.x_in.shape[1] + 3 * 4 * M

    def d2h_bytes(self, M: int) -> int:
        return 4 * (3 + M) + 2 * M * self.y_down_red.shape[1]


class _Eager:
    """replay() = one eager forward (VerifyStack.capture when the process group cannot be captured)."""

    def __init__(self, st: "VerifyStack", M: int):
        self.st, self.M = st, M

    def replay(self):
        self.st.forward(self.M)


def _peer_group(nbytes: int, slots: int, group):
    """The symmetric regions of a fused all-reduce: CUDA-IPC peer mappings (verified: simulated ranks, two
    processes); with W4A16_NVLS=1 first an NVLS multicast object (multimem loads / reds), which no box of this
    build could create yet, so it is opt-in. Every step is agreed on by all ranks, so a failure anywhere falls
    back everywhere (e.g. several ranks on one GPU cannot share a multicast object)."""
    import os
    if os.environ.get("W4A16_NVLS") == "1":
        try:
            return PeerGroup.mc(nbytes, slots, group)
        except W4A16Error:
            pass
    return PeerGroup.ipc(nbytes, slots, group)


class _Calibration:
    """Build-time weight scaling of VerifyStack(calibrate=x0): runs the forward's data flow op by op from x0
    through the layers as they are built (libw4a16 kernels; torch only for the RMS reduction and the scalar
    multiply) and scales each weight by 1 / RMS of its output before packing it for good."""

    def __init__(self, st: "VerifyStack", x0: torch.Tensor):
        self.st = st
        self.M = x0.shape[0]
        P = st.plan
        self.ws = alloc_workspace(self.M, [(s["K"], s["N"]) for s in P.values()], device=st.device)
        self.h = x0.to(st.device).contiguous().clone()
        self.q = self.o = self.act = None

    def _rms(self, y: torch.Tensor, column_parallel: bool) -> float:
        st = self.st
        if st.t > 1 and not column_parallel:      # row-parallel: the model's output is the reduced sum
            dist.all_reduce(y, group=st.group)
        ss = torch.stack([(y.float() ** 2).sum(), torch.tensor(float(y.numel()), device=y.device)])
        if st.t > 1 and column_parallel:          # column shards: RMS over the full output
            dist.all_reduce(ss, group=st.group)
        return float((ss[0] / ss[1]).sqrt().item())

    def step(self, l: int, name: str, W: torch.Tensor, pl):
        st, M = self.st, self.M
        X = {"qkv": self.h, "o": self.q, "gate_up": self.o, "down": self.act}[name]
        y = torch.empty(M, pl.N, dtype=torch.float16, device=st.device)
        col = name in ("qkv", "gate_up")
        pl(X, y, self.ws)
        r = self._rms(y, col)
        # a power of two: the scaled fp16 weight is exact (reproducible bit for bit on the host) and the
        # output RMS lands in [1/sqrt(2), sqrt(2)] — each op is calibrated on its actual input, so it does
        # not compound over the layers
        alpha = 2.0 ** round(-math.log2(r)) if r > 0 and math.isfinite(r) else 1.0
        W.mul_(alpha)
        pl = pack_linear(W, mode=st.mode, dev_status=st.status)
        pl(X, y, self.ws)
        if not col and st.t > 1:
            dist.all_reduce(y, group=st.group)
        while len(st.calib_scale) <= l:
            st.calib_scale.append({})
        st.calib_scale[l][name] = alpha
        if name == "qkv":
            self.q = y[:, : st.plan["o"]["K"]].contiguous()
        elif name == "o":
            self.o = y
        elif name == "gate_up":
            self.act = torch.empty(M, st.plan["down"]["K"], dtype=torch.float16, device=st.device)
            w4a16_silu_mul_blocked(y, self.act, SILU_BLOCK)
        else:
            self.h = y
        return pl
