#!/usr/bin/env python
"""Benchmark of the W4A16 verify hot path (BASELINE.json metric: "W4A16 verify-GEMM µs and achieved HBM
TB/s vs draft width M=1-64").

Step = one verify forward of the Llama-3-70B W4A16 linear stack (80 decoder layers: QKV, O, gate-up,
SiLU*mul, down; attention/norms out of scope) at draft width M, then greedy acceptance of an M-node draft
tree (BASELINE.json configs 3-5; config 4 at N GPUs = tensor-parallel over N ranks with NCCL all-reduce).
value = algorithmic weight bytes streamed by all ranks per step / max-over-ranks step time, in TB/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--M 8] [--layers 80] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Inputs are seeded synthetic (synth/), resident in HBM before timing; per-step weights (36.4 GB at N=1)
exceed the 126 MB L2, so no flush is needed between steps. Timing: CUDA graph replays bracketed by CUDA
events on the launching stream, barrier + synchronize on both sides, max over ranks.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "W4A16 verify-GEMM µs and achieved HBM TB/s vs draft width M=1–64"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
TAU = {  # paper accepted lengths for config 5 (PAPER.md lines)
    "eagle2_d6_n48": (49, 3.81, "P:757"),
    "eagle2_n60_tree": (61, 3.81, "P:757 (tau of the d=6 tree; BASELINE config 5 tree of 60)"),
    "vanilla_sp_d6": (7, 4.72, "P:714"),
    "vanilla_sp_d7": (8, 5.09, "P:722"),
    "hierspec_6_3": (7, 5.28, "P:768"),
    "hierspec_7_3": (8, 5.46, "P:784"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--M", type=int, default=8, help="headline draft width (verify rows): 8 = HierSpec's 70B sequence "
                    "verification d = 7 (P:784), M = d + 1 (reading R10)")
    ap.add_argument("--layers", type=int, default=None, help="decoder layers (default: the model's)")
    ap.add_argument("--model", default="70b", choices=["70b", "8b"])
    ap.add_argument("--mode", default="asym", choices=["asym", "sym"])
    ap.add_argument("--sweep", default="1,2,4,7,8,16,24,32,49,61,64", help="comma list of M for the M sweep ('' = none)")
    ap.add_argument("--sweep-steps", type=int, default=10)
    ap.add_argument("--windows", type=int, default=3, help="timed windows of --steps replays; the headline is their median")
    ap.add_argument("--sym-sweep", default="1,8,16,64", help="M sweep of the same stack in the paper's own GPTQ "
                    "symmetric format (P:103; '' = none)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--allreduce", default="auto", choices=["auto", "nccl", "fused"],
                    help="tp > 1: ALLREDUCE ops inside one chain per forward over CUDA-IPC peer memory (fused, "
                         "include/w4a16.h) or NCCL all-reduces between per-segment chains; auto = fused if its "
                         "setup and a start-up check against the NCCL path pass on every rank, else nccl")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-kernels", dest="kernels", action="store_false", help="skip the per-kernel breakdown")
    ap.add_argument("--no-lm-head", dest="lm_head", action="store_false",
                    help="skip the LM head + argmax measurement (SURVEY 8(f) f3)")
    return ap.parse_args()


_T0 = time.perf_counter()


def log(msg):
    """Progress on stderr (the JSON line is the only stdout output)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# --------------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------------------------------
# CPU baseline: the oracle as it stands, on a bounded sample of the workload
# --------------------------------------------------------------------------------------------------
_SAMPLE = {}
SHAPES_70B = {"qkv": (8192, 10240), "o": (8192, 8192), "gate_up": (8192, 57344), "down": (28672, 8192)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _slice_inputs(K, N, M, seed):
    """Oracle inputs for a K x N W4A16 GEMM at width M, built once (untimed, like the GPU arm's resident
    inputs): codes uniform in [0, 15], per-group fp16 scales / zeros, seeded activations. The oracle's cost
    does not depend on the values, so the codes come from numpy instead of quantising generated weights."""
    import numpy as np

    import synth
    key = (K, N, M, seed)
    if key not in _SAMPLE:
        rng = np.random.default_rng(seed + K + 7 * N)
        codes = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
        sc = np.full((K // 128, N), np.float16(0.0023).view(np.uint16), dtype=np.uint16)
        ze = rng.integers(0, 16, size=(K // 128, N)).astype(np.float16).view(np.uint16)
        X = synth.host(seed, 9002 + K, synth.ACT, M, K)
        _SAMPLE[key] = (X, codes, sc, ze)
    return _SAMPLE[key]


def _tree(M, seed):
    import numpy as np

    import synth
    rng = np.random.default_rng(seed)
    tok, par = synth.eagle_tree(rng, max(M - 1, 0), 6)
    return tok, par, synth.target_argmax_for(rng, tok, par, 0.7)


def oracle_layer_slice(M, seed, den=64, threads=None):
    """Time the oracle on one Llama-3-70B decoder layer restricted to 1/den of every matrix's output columns
    (QKV, O, gate-up, down) at width M, plus oracle.accept on an M-node tree. Returns (TB/s of the slice's
    W4 weight bytes, seconds, sample text, threads). The per-column cost is uniform, so this is the layer's
    throughput on this host."""
    import oracle
    threads = threads or (os.cpu_count() or 1)
    ins = [(_slice_inputs(K, N // den, M, seed), K, N // den) for K, N in SHAPES_70B.values()]
    tok, par, am = _tree(M, seed)
    t0 = time.perf_counter()
    for (X, c, sc, ze), K, N in ins:
        oracle.gemm(X, c, sc, ze, nthreads=threads)
    oracle.accept(tok, par, am)
    dt = time.perf_counter() - t0
    wbytes = sum(K * N // 2 + (K // 128) * N * 4 for _, K, N in ins)
    sample = (f"oracle.gemm (fp64) on one Llama-3-70B layer restricted to 1/{den} of each matrix's output columns "
              f"({wbytes / 1e6:.2f} MB of W4 weights) at M={M} + oracle.accept on a {M}-node tree, {threads} threads")
    return wbytes / dt / 1e12, dt, sample, threads


def cpu_baseline_plan(M_head, seed):
    """BASELINE.md's CPU-baseline plan: config 1 on 1 thread and on all host threads; one 70B
    layer at M in {1, M_head, 64} on all threads (timed on a column slice, per-column cost uniform),
    extrapolated x80 to the stack and labelled so; the CPU model string."""
    import oracle
    threads = os.cpu_count() or 1
    out = {"cpu_model": cpu_model(), "nproc": threads}
    X, c, sc, ze = _slice_inputs(4096, 4096, 8, seed)
    tok8 = [100, 11, 12, 21, 22, 23, 31, 32]
    par8 = [-1, 0, 0, 1, 1, 2, 3, 5]
    am8 = [12, 99, 23, 31, 99, 32, 99, 40]
    c1 = {}
    for th in sorted({1, threads}):
        t0 = time.perf_counter()
        oracle.gemm(X, c, sc, ze, nthreads=th)
        oracle.accept(tok8, par8, am8)
        c1[f"threads_{th}"] = {"s": time.perf_counter() - t0}
    wb1 = 4096 * 4096 // 2 + 32 * 4096 * 4
    for v in c1.values():
        v["TBps"] = wb1 / v["s"] / 1e12
    out["config1_gemm4096_M8_plus_accept8"] = c1
    layer = {}
    for M in sorted({1, M_head, 64}):
        v, dt, sample, th = oracle_layer_slice(M, seed, den=32, threads=threads)
        per_layer = dt * 32
        layer[str(M)] = {"TBps": v, "s_per_layer": per_layer, "s_per_80_layer_forward_extrapolated": 80 * per_layer,
                         "timed_on": "1/32 of every matrix's output columns (x32 for the layer, x80 for the stack)"}
    out["llama3_70b_layer"] = layer
    return out


def run_reference(args):
    """--impl reference: the task's reference arm for this tier = the oracle as it stands on the host cores,
    each step a bounded sample of the same workload (one 70B layer on 1/64 of its columns at width M)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    M = args.M
    for _ in range(args.warmup):
        oracle_layer_slice(M, args.seed)
    times, wbytes, sample, threads = [], None, "", 1
    for _ in range(args.steps):
        v, dt, sample, threads = oracle_layer_slice(M, args.seed)
        times.append(dt)
        wbytes = v * dt * 1e12
    tot = sum(times)
    value = wbytes * len(times) / tot / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"llama3-70b W4A16 g128 {args.mode} verify forward: 80 decoder layers (QKV, O, gate-up, "
                               f"SiLU*mul, down) + verify_accept; BASELINE configs 3-4", "M": M, "layers": 80, "tp": args.gpus,
                   "parallelism": f"tp{args.gpus}",
                   "timing": "the oracle on a bounded sample of this workload (see cpu_baseline.sample), host cores"},
        "cpu_baseline": {"value": value, "unit": "TB/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "TB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------------
def main():
    args = parse()
    if os.environ.get("BENCH_WATCHDOG"):   # diagnostics: dump the Python stack if the run stalls
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["BENCH_WATCHDOG"]), exit=True)
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2505_22179_b200 as w4
    import synth
    from paper_2505_22179_b200 import tp

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # BENCH_DIST_BACKEND=gloo (tests only): the control plane over gloo and every rank on cuda:(local % #GPUs),
    # so the multi-rank code path (fused all-reduce set-up, start-up check, NCCL fallback) runs on a 1-GPU box
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD

    def dist_barrier():
        if backend == "nccl":
            dist.barrier(device_ids=[local])
        else:
            dist.barrier()
    dims = tp.LLAMA3_70B if args.model == "70b" else tp.LLAMA3_8B
    n_layers = args.layers or dims.layers
    mode = w4.W4A16_SYM if args.mode == "sym" else w4.W4A16_ASYM
    sweep = [int(x) for x in args.sweep.split(",") if x.strip()]
    M_max = max([args.M] + sweep)
    mat_id = {n: i for i, n in enumerate(tp.MATRICES)}

    def make_weight(l, name, K, N, out):
        synth.gpu(args.seed, synth.tensor_id(l, mat_id[name], rank), synth.WEIGHT, K, N, out=out)

    def build(allreduce, mode=mode):
        # weights scaled at build time (powers of two) so every GEMM output keeps O(1) RMS along the forward's
        # data flow (tp.py: the norms are outside the hot path); the same calibration input on every rank
        x0 = synth.gpu(args.seed, synth.tensor_id(0xFFF, 9, 0), synth.ACT, 8, dims.hidden)
        st = tp.VerifyStack(dims, n_layers, M_max, make_weight, tp_size=world, tp_rank=rank, group=group, mode=mode,
                            device=dev, allreduce=allreduce, calibrate=x0)
        # the forward's input hidden state (seeded, in HBM, identical on every rank) and a draft tree
        synth.gpu(args.seed, synth.tensor_id(0xFFF, 1, 0), synth.ACT, st.x_in.shape[0], st.x_in.shape[1], out=st.x_in)
        rng = np.random.default_rng(args.seed)
        tok, par = synth.eagle_tree(rng, M_max - 1, 6)
        am = synth.target_argmax_for(rng, tok, par, 0.7)
        st.set_tree(tok, par, am)
        torch.cuda.synchronize()
        return st

    def fused_matches_nccl(st) -> bool:
        """One forward at M = min(8, M_max) through the fused chain vs the same forward op by op with NCCL."""
        m = min(8, M_max)
        dist_barrier()
        st.forward(m)
        torch.cuda.synchronize()
        got = [st.y_o_red[:m].float().clone(), st.y_down_red[:m].float().clone()]
        st.use_chains = False
        st.forward(m)
        torch.cuda.synchronize()
        st.use_chains = True
        want = [st.y_o_red[:m].float(), st.y_down_red[:m].float()]
        if os.environ.get("BENCH_FAIL_FUSED_CHECK") == str(rank):   # tests only: exercise the fallback branch
            return False
        return all(bool(torch.all((g - w).abs() <= 1e-2 * (1 + w.abs())).item()) for g, w in zip(got, want))

    t0 = time.perf_counter()
    allreduce_used = "none" if world == 1 else args.allreduce
    stack = None
    if world > 1 and args.allreduce in ("auto", "fused"):
        ok = True
        try:
            stack = build("fused")
            ok = fused_matches_nccl(stack)
        except Exception as e:   # setup failure (IPC / peer access): every rank learns it below
            log(f"fused all-reduce unavailable on rank {rank}: {e!r}")
            ok = False
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            allreduce_used = f"fused ({stack.peers.kind})"   # NVLS multicast or peer-load regions
        elif args.allreduce == "fused":
            raise SystemExit("--allreduce fused: setup or start-up check failed")
        else:
            log(f"falling back to {backend} all-reduces")
            stack = None   # its peer region stays mapped (a few MB): freeing it needs every peer to unmap first
            torch.cuda.empty_cache()
            allreduce_used = backend
    if stack is None:
        stack = build("nccl")
    # gloo (tests only) cannot be captured in a CUDA graph: its process-group all-reduces run eagerly
    stack.capturable = backend == "nccl" or world == 1 or allreduce_used.startswith("fused")
    build_s = time.perf_counter() - t0
    log(f"built {n_layers} layers ({stack.weight_bytes / 1e9:.2f} GB packed) in {build_s:.1f}s, all-reduce: {allreduce_used}")

    def barrier():
        if world > 1:
            dist_barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.Stream(dev)

    def time_graph(g, steps, warmup, windows=1):
        """ms per step: `windows` timed windows of exactly `steps` replays each (barrier + synchronize on both
        sides, CUDA events on the launching stream, max over ranks); the median window is returned."""
        with torch.cuda.stream(stream):
            for _ in range(warmup):
                g.replay()
        res = []
        for _ in range(windows):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(steps):
                    g.replay()
                e1.record(stream)
            barrier()
            res.append(max_over_ranks(e0.elapsed_time(e1)) / steps)
        time_graph.windows = res
        return statistics.median(res)

    clocks = ClockSampler(local) if rank == 0 else None
    bytes_all_ranks = stack.weight_bytes * world  # shards partition the model: == full model bytes
    gH = stack.capture(args.M)
    log(f"captured M={args.M}")
    ms = time_graph(gH, args.steps, args.warmup, windows=args.windows)
    windows_ms = list(time_graph.windows)
    log(f"headline M={args.M}: {ms:.3f} ms/step (median of {args.windows} windows: "
        + ", ".join(f"{w:.3f}" for w in windows_ms) + ")")
    # per-step distribution (median and p10/p90 over replays), events around every replay
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with torch.cuda.stream(stream):
        ev[0].record(stream)
        for i in range(args.steps):
            gH.replay()
            ev[i + 1].record(stream)
    torch.cuda.synchronize()
    per_step = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))
    pct = lambda q: per_step[min(len(per_step) - 1, int(q * (len(per_step) - 1) + 0.5))]
    step_dist = {"p10": pct(0.1), "p50": pct(0.5), "p90": pct(0.9), "n": len(per_step)}
    value = bytes_all_ranks / (ms * 1e-3) / 1e12

    # M sweep (same protocol)
    m_sweep = {}
    for M in sweep:
        g = stack.capture(M)
        msM = time_graph(g, args.sweep_steps, 3)
        log(f"sweep M={M}: {msM:.3f} ms/forward")
        m_sweep[str(M)] = {"ms_per_forward": msM, "us_per_layer": 1e3 * msM / n_layers,
                           "TBps": bytes_all_ranks / (msM * 1e-3) / 1e12}
    peak_gbs, peak_src = hbm_peak()
    for v in m_sweep.values():
        v["frac_hbm"] = v["TBps"] * 1e3 / (peak_gbs * world)
    if "1" in m_sweep and "64" in m_sweep:
        ratio_64 = m_sweep["64"]["ms_per_forward"] / m_sweep["1"]["ms_per_forward"]
    else:
        ratio_64 = None
    # the same stack in the paper's own weight format, GPTQ symmetric g128 (z = 8, no zero bytes)
    sym_sweep = None
    sym_ms = [int(x) for x in args.sym_sweep.split(",") if x.strip()] if args.mode == "asym" else []
    if sym_ms:
        try:
            st_sym = build("nccl", mode=w4.W4A16_SYM)
            bs = st_sym.weight_bytes * world
            sym_sweep = {"weight_bytes_per_step": bs, "format": "GPTQ symmetric g128 (z = 8): 0.515625 B/weight"}
            for M in sym_ms:
                msM = time_graph(st_sym.capture(M), args.sweep_steps, 3)
                sym_sweep[str(M)] = {"ms_per_forward": msM, "TBps": bs / (msM * 1e-3) / 1e12,
                                     "frac_hbm": bs / (msM * 1e-3) / 1e9 / (hbm_peak()[0] * world)}
                log(f"SYM sweep M={M}: {msM:.3f} ms/forward")
            del st_sym
            torch.cuda.empty_cache()
        except Exception as e:   # never let the side measurement break the bench line
            sym_sweep = {"error": repr(e)}
    hier = {}
    for k, (M, tau, cite) in TAU.items():
        if str(M) in m_sweep:
            hier[k] = {"M": M, "tau": tau, "cite": cite, "us_per_token": 1e3 * m_sweep[str(M)]["ms_per_forward"] / tau}

    # e2e through the public API: pinned host inputs -> device -> forward -> accept result + hidden -> host
    M = args.M
    pin = dict(pin_memory=True)
    host_in = {"x_in": stack.x_in.cpu().pin_memory(), "tokens": stack.tokens.cpu().pin_memory(),
               "parents": stack.parents.cpu().pin_memory(), "argmax": stack.argmax.cpu().pin_memory()}
    host_out = {"accept": torch.empty(3 + M_max, dtype=torch.int32, **pin),
                "y": torch.empty(M_max, stack.y_down.shape[1], dtype=torch.float16, **pin)}
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            stack.verify_host(M, host_in, host_out, gH)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            stack.verify_host(M, host_in, host_out, gH)
        e1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    log(f"e2e: {ms_e2e:.3f} ms/step")
    acc = host_out["accept"][:3].tolist()

    # per-kernel breakdown: each GEMM kind back-to-back over all layers (distinct weights), one graph each
    kernels = {}
    roofline = None
    if args.kernels:
        P = stack.plan
        for name in tp.MATRICES:
            s = P[name]
            xin = {"qkv": stack.x_in[:M], "o": stack.q_part(M), "gate_up": stack.y_o_red[:M], "down": stack.act[:M]}[name]
            yout = {"qkv": stack.y_qkv, "o": stack.y_o, "gate_up": stack.y_gu, "down": stack.y_down}[name][:M]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                for L in stack.layers:
                    L[name](xin, yout, stack.ws, stream)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for L in stack.layers:
                    L[name](xin, yout, stack.ws, stream)
            msk = time_graph(g, max(3, args.steps // 2), 2) / n_layers
            log(f"kernel {name}: {1e3 * msk:.2f} us")
            wb = stack.layers[0][name].weight_bytes
            kernels[name] = {"K": s["K"], "N": s["N"], "us": 1e3 * msk, "weight_MB": wb / 1e6,
                             "GBps": wb / (msk * 1e-3) / 1e9, "frac_hbm": wb / (msk * 1e-3) / 1e9 / peak_gbs,
                             "family": w4.w4a16_gemm_family(M, s["K"], s["N"])}
            # the other engine (mma.sync <-> tcgen05) on the same launches, for comparison (not part of the step)
            alt = (w4.W4A16_FAMILY_TCGEN05 if kernels[name]["family"] != w4.W4A16_FAMILY_TCGEN05 else
                   w4.W4A16_FAMILY_MMA_SYNC if M <= 16 else None)
            if alt is None:
                continue
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                for L in stack.layers:
                    L[name](xin, yout, stack.ws, stream, family=alt)
            torch.cuda.synchronize()
            with torch.cuda.graph(g2, stream=stream):
                for L in stack.layers:
                    L[name](xin, yout, stack.ws, stream, family=alt)
            msa = time_graph(g2, max(3, args.steps // 2), 2) / n_layers
            kernels[name]["other_family"] = {"family": alt, "us": 1e3 * msa, "GBps": wb / (msa * 1e-3) / 1e9}
            del g2
        gate = kernels["gate_up"]
        chains = stack.chains(M) if stack.use_chains else None
        if chains is not None:
            # dominant kernel = the persistent chain: the whole verify forward (tp = 1) or one segment
            gc = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                for c in chains:
                    c(stream)
            torch.cuda.synchronize()
            with torch.cuda.graph(gc, stream=stream):
                for c in chains:
                    c(stream)
            msc = time_graph(gc, max(3, args.steps // 2), 2) / len(chains)
            del gc
            per_launch = stack.weight_bytes / len(chains)
            act_bytes = sum(2 * M * (s["K"] + s["N"]) for s in P.values()) * n_layers // len(chains)
            log(f"chain kernel: {msc:.3f} ms per launch")
            roofline = {"bound": "hbm", "kernel": f"w4a16 chain kernel ({len(chains)} launch(es) per forward, "
                                                  f"{stack.chains(M)[0].n} ops per launch, M={M})",
                        "achieved": per_launch / (msc * 1e-3) / 1e9, "peak": peak_gbs, "unit": "GB/s",
                        "frac": per_launch / (msc * 1e-3) / 1e9 / peak_gbs, "traffic": None, "peak_source": peak_src,
                        "algorithmic_bytes_per_launch": per_launch + act_bytes,
                        "note": "achieved = packed weight bytes per launch / its average duration (CUDA events on the "
                                "launching stream over back-to-back graph replays); activation bytes (L2-resident) "
                                "listed but not counted"}
            fam_tag = f"chain_M{M}"
        else:
            roofline = {"bound": "hbm", "kernel": f"w4a16 GEMM gate-up (K={gate['K']}, N={gate['N']}, M={M})",
                        "achieved": gate["GBps"], "peak": peak_gbs, "unit": "GB/s", "frac": gate["GBps"] / peak_gbs,
                        "traffic": None, "peak_source": peak_src,
                        "algorithmic_bytes_per_launch": stack.layers[0]["gate_up"].weight_bytes + 2 * M * (gate["K"] + gate["N"]),
                        "note": "achieved = weight bytes/launch / avg launch time over 80 back-to-back launches (CUDA "
                                "graph, CUDA events on the launching stream)"}
            fam_tag = ("famB" if gate["family"] == w4.W4A16_FAMILY_TCGEN05 else "famA") + f"_gateup_M{M}"
        ncu_path = next((q for q in (os.path.join(ROOT, "profiles", f"r{r:02d}_ncu_{fam_tag}.json") for r in (2, 1))
                         if os.path.exists(q)), "")   # the newest round's committed capture
        if os.path.exists(ncu_path):   # committed ncu --set full capture of this kernel at this M
            try:
                with open(ncu_path) as f:
                    d = json.load(f)["derived"]
                # the capture may cover a shorter stack (the chain capture is 8 layers): DRAM bytes per packed
                # weight byte from ncu, times this launch's packed weight bytes
                per_w = d["dram_traffic_bytes"] / d["algorithmic_bytes"]
                w_launch = stack.weight_bytes / len(chains) if chains is not None else stack.layers[0]["gate_up"].weight_bytes
                roofline["traffic"] = per_w * w_launch
                roofline["traffic_over_weight_bytes"] = per_w
                roofline["traffic_source"] = os.path.relpath(ncu_path, ROOT) + " (dram__bytes_read.sum + dram__bytes_write.sum, scaled per weight byte)"
            except Exception:
                pass
    # BASELINE configs 1 and 2 beside the headline (config 3-4): a single 4096x4096 W4A16 GEMM at M=8 with
    # acceptance on the 8-node tree (config 1), and the Llama-3-8B linear stack's M sweep (config 2).
    other_configs = None
    if args.lm_head and rank == 0 and world == 1:
        other_configs = {}
        R1 = 64   # distinct 4096x4096 weights back to back (64 x 8.9 MB >> L2)
        lins = []
        for r in range(R1):
            Wt = synth.gpu(args.seed, synth.tensor_id(0xFFC, r, 0), synth.WEIGHT, 4096, 4096)
            lins.append(w4.pack_linear(Wt))
            del Wt
        X1 = synth.gpu(args.seed, synth.tensor_id(0xFFC, 255, 0), synth.ACT, 8, 4096)
        Y1 = torch.empty(8, 4096, dtype=torch.float16, device=dev)
        ws1 = w4.alloc_workspace(8, [(4096, 4096)], device=dev)
        tok8 = torch.tensor([100, 11, 12, 21, 22, 23, 31, 32], dtype=torch.int32, device=dev)
        par8 = torch.tensor([-1, 0, 0, 1, 1, 2, 3, 5], dtype=torch.int32, device=dev)
        am8 = torch.tensor([12, 99, 23, 31, 99, 32, 99, 40], dtype=torch.int32, device=dev)
        out8 = torch.empty(11, dtype=torch.int32, device=dev)
        with torch.cuda.stream(stream):
            for l in lins:
                l(X1, Y1, ws1, stream)
            w4.verify_accept(tok8, par8, am8, out8, stream=stream)
        torch.cuda.synchronize()
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=stream):
            for l in lins:
                l(X1, Y1, ws1, stream)
        ms1 = time_graph(g1, 5, 2) / R1
        ga = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga, stream=stream):
            for _ in range(50):
                w4.verify_accept(tok8, par8, am8, out8, stream=stream)
        msa = time_graph(ga, 5, 2) / 50
        wb1 = lins[0].weight_bytes
        # the same 64 independent GEMMs (same X, own Y each) as ONE persistent chain launch: no per-launch ramp,
        # no dependency between them — the steady-state per-GEMM cost of the kernel at this size
        Ys = torch.empty(R1, 8, 4096, dtype=torch.float16, device=dev)
        chb = w4.Chain([("gemm", X1, l, Ys[r]) for r, l in enumerate(lins)], 8)
        with torch.cuda.stream(stream):
            chb(stream)
        torch.cuda.synchronize()
        gb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gb, stream=stream):
            chb(stream)
        msb = time_graph(gb, 5, 2) / R1
        other_configs["config1_gemm4096_M8"] = {"us": 1e3 * ms1, "TBps": wb1 / (ms1 * 1e-3) / 1e12,
                                                "frac_hbm": wb1 / (ms1 * 1e-3) / 1e9 / peak_gbs,
                                                "accept_8node_us": 1e3 * msa,
                                                "note": "64 distinct weights back to back in a CUDA graph, one launch each",
                                                "batched_in_one_chain": {
                                                    "us": 1e3 * msb, "TBps": wb1 / (msb * 1e-3) / 1e12,
                                                    "frac_hbm": wb1 / (msb * 1e-3) / 1e9 / peak_gbs,
                                                    "note": "the same 64 independent GEMMs as one persistent chain launch"}}
        log(f"config 1 batched in one chain: {1e3 * msb:.2f} us per GEMM")
        del lins, g1, ga, gb, chb, Ys
        log(f"config 1: {1e3 * ms1:.2f} us per 4096x4096 GEMM at M=8, accept {1e3 * msa:.2f} us")
        d8 = tp.LLAMA3_8B

        def make8(l, name, K, N, out):
            synth.gpu(args.seed, synth.tensor_id(l, mat_id[name], 0xEE), synth.WEIGHT, K, N, out=out)

        st8 = tp.VerifyStack(d8, d8.layers, 64, make8, device=dev,
                             calibrate=synth.gpu(args.seed, synth.tensor_id(0xFFB, 9, 0), synth.ACT, 8, d8.hidden))
        synth.gpu(args.seed, synth.tensor_id(0xFFB, 1, 0), synth.ACT, 64, d8.hidden, out=st8.x_in)
        sw8 = {}
        for M8 in (1, 4, 8, 16, 32, 64):
            g8 = st8.capture(M8)
            ms8 = time_graph(g8, 10, 3)
            sw8[str(M8)] = {"ms_per_forward": ms8, "TBps": st8.weight_bytes / (ms8 * 1e-3) / 1e12,
                            "frac_hbm": st8.weight_bytes / (ms8 * 1e-3) / 1e9 / peak_gbs}
        other_configs["config2_llama3_8b_sweep"] = {"layers": d8.layers, "weight_bytes": st8.weight_bytes,
                                                    "m_sweep": sw8}
        log("config 2 (8B) sweep: " + ", ".join(f"M={k}: {v['ms_per_forward']:.3f} ms" for k, v in sw8.items()))
        del st8
        torch.cuda.empty_cache()
    # FP16 LM head [M, hidden] x [hidden, vocab] with the greedy argmax fused (the target_argmax
    # that verify_accept consumes), measured on its own: its weights (2.1 GB fp16) are not W4A16 bytes.
    lm = None
    if args.lm_head and rank == 0:
        V = 128256
        Kh = dims.hidden
        R = 3   # distinct heads back to back (3 x 2.1 GB >> L2)
        heads = [synth.gpu(args.seed, synth.tensor_id(0xFFE, r, 0), synth.WEIGHT, V, Kh) for r in range(R)]
        hid = stack.y_down[:M] if stack.y_down.shape[1] == Kh else torch.zeros(M, Kh, dtype=torch.float16, device=dev)
        am = torch.empty(M, dtype=torch.int32, device=dev)
        mx = torch.empty(M, dtype=torch.float32, device=dev)
        lws = w4.alloc_lmhead_workspace(M, Kh, V, device=dev)
        with torch.cuda.stream(stream):
            for h in heads:
                w4.w4a16_lmhead_argmax(hid, h, am, lws, out_max=mx, stream=stream)
        torch.cuda.synchronize()
        gl = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gl, stream=stream):
            for h in heads:
                w4.w4a16_lmhead_argmax(hid, h, am, lws, out_max=mx, stream=stream)
        msl = time_graph(gl, 5, 2) / R
        hb = V * Kh * 2
        lm = {"row": "f3", "what": f"FP16 LM head {Kh}x{V} + fused greedy argmax at M={M} (w4a16_lmhead_argmax)",
              "us": 1e3 * msl, "GBps": hb / (msl * 1e-3) / 1e9, "frac_hbm": hb / (msl * 1e-3) / 1e9 / peak_gbs,
              "weight_bytes": hb, "bound": "hbm"}
        log(f"lm head + argmax: {1e3 * msl:.1f} us ({lm['frac_hbm']:.2f} of HBM)")
        del heads, gl
    # tree-masked verify attention over a 2048-token cached prefix (Llama-3-70B: 64 q heads,
    # 8 kv heads, head 128) at the headline width (sequence draft) and at the BASELINE config-5 tree of 60
    # drafts, plus the KV compaction that follows acceptance; per layer (x80 for the forward).
    attn = None
    if args.lm_head and rank == 0:
        Lctx, Hq, Hkv, D = 2048, dims.n_q // world, dims.n_kv // world, dims.head
        attn = {"row": "f2", "context": Lctx, "heads": [Hq, Hkv, D]}
        for Mq, kind in ((M, "sequence"), (61, "eagle2_tree_60")):
            Qa = synth.gpu(args.seed, synth.tensor_id(0xFFD, 1, Mq), synth.ACT, Mq, Hq * D).view(Mq, Hq, D)
            Ka = synth.gpu(args.seed, synth.tensor_id(0xFFD, 2, Mq), synth.ACT, Lctx + Mq, Hkv * D).view(Lctx + Mq, Hkv, D)
            Va = synth.gpu(args.seed, synth.tensor_id(0xFFD, 3, Mq), synth.ACT, Lctx + Mq, Hkv * D).view(Lctx + Mq, Hkv, D)
            if kind == "sequence":
                par_a = torch.arange(-1, Mq - 1, dtype=torch.int32, device=dev)
            else:
                _, pa = synth.eagle_tree(np.random.default_rng(args.seed), Mq - 1, 6)
                par_a = torch.tensor(pa, dtype=torch.int32, device=dev)
            Oa = torch.empty(Mq, Hq, D, dtype=torch.float16, device=dev)
            wsa = torch.zeros(w4.w4a16_tree_attention_workspace_bytes(Mq, Lctx, Hq, Hkv, D), dtype=torch.uint8, device=dev)
            acc_a = torch.zeros(3 + Mq, dtype=torch.int32, device=dev)
            with torch.cuda.stream(stream):
                w4.w4a16_tree_attention(Qa, Ka, Va, par_a, Oa, wsa, stream=stream)
            torch.cuda.synchronize()
            ga = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ga, stream=stream):
                for _ in range(20):
                    w4.w4a16_tree_attention(Qa, Ka, Va, par_a, Oa, wsa, stream=stream)
            msa = time_graph(ga, 5, 2) / 20
            kv_bytes = 2 * (Lctx + Mq) * Hkv * D * 2
            attn[kind] = {"M": Mq, "us_per_layer": 1e3 * msa, "kv_GBps": kv_bytes / (msa * 1e-3) / 1e9,
                          "us_per_forward_80_layers": 80 * 1e3 * msa}
            log(f"tree attention M={Mq} ({kind}): {1e3 * msa:.1f} us per layer")
            del ga
    # the in-chain ALLREDUCE op's own cost on one GPU — a world-1 group (tile counters bumped by
    # the O / down GEMMs' tile writers, system fences, per-tile reduce; no NVLink reads): 16 layers as one
    # chain with and without an ALLREDUCE after every O and down GEMM, over a peer-load group and (where the
    # device supports multicast objects) an NVLS group.
    ar = None
    if args.lm_head and world == 1 and M <= 16 and n_layers >= 16:
        try:
            nl = 16
            Hd = dims.hidden
            kinds = ["peer"] + (["nvls"] if w4.PeerGroup.mc_supported() else [])
            t_ch, groups = {}, {}
            nvls_error = "device reports no multicast support"
            plain = []
            for l, L in enumerate(stack.layers[:nl]):
                qa, qb = stack._layer_ops(L, M, l)
                plain += qa + qb
            cases = [("plain", plain)]
            for kind in list(kinds):
                try:
                    g1 = (w4.PeerGroup.simulated(1, 1 << 22, 2 * nl, device=dev)[0] if kind == "peer" else
                          w4.PeerGroup.mc(1 << 22, 2 * nl))
                except w4.W4A16Error as e:   # multicast objects refused on this device (e.g. a GPU partition)
                    kinds.remove(kind)
                    nvls_error = repr(e)
                    continue
                groups[kind] = g1
                P_o, P_d = g1.alloc(M, Hd), g1.alloc(M, Hd)
                r_o, r_d = (torch.empty(M, Hd, dtype=torch.float16, device=dev) for _ in range(2))
                fused = []
                for l, L in enumerate(stack.layers[:nl]):
                    h = stack.x_in[:M] if l == 0 else r_d
                    fused += [("gemm", h, L["qkv"], stack.y_qkv[:M]), ("gemm", stack.q_part(M), L["o"], P_o),
                              ("allreduce", P_o, r_o, g1), ("gemm_silu", r_o, L["gate_up"], stack.act[:M]),
                              ("gemm", stack.act[:M], L["down"], P_d), ("allreduce", P_d, r_d, g1)]
                cases.append((kind, fused))
            for name, ops in cases:
                ch = w4.Chain(ops, M)
                with torch.cuda.stream(stream):
                    ch(stream)
                torch.cuda.synchronize()
                gch = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gch, stream=stream):
                    ch(stream)
                t_ch[name] = time_graph(gch, 10, 3)
                del gch, ch
            ar = {"row": "f1", "M": M, "layers": nl, "ops": 2 * nl, "world": 1, "chain_ms": t_ch["plain"],
                  "nvls": "measured" if "nvls" in kinds else f"unavailable: {nvls_error}",
                  "note": "world-1 group on one GPU: fused per-tile protocol (tile counters, system fences, per-tile "
                          "reduce); NVLink reads not included"}
            for kind in kinds:
                ar[f"chain_with_allreduce_ms_{kind}"] = t_ch[kind]
                ar[f"us_per_allreduce_op_{kind}"] = 1e3 * (t_ch[kind] - t_ch["plain"]) / (2 * nl)
                log(f"in-chain ALLREDUCE (world 1, {kind}): {ar[f'us_per_allreduce_op_{kind}']:.2f} us per op")
            ar["us_per_allreduce_op"] = ar["us_per_allreduce_op_peer"]
            for g1 in groups.values():
                g1.close()
        except Exception as e:   # never let the side measurement break the bench line
            ar = {"row": "f1", "error": repr(e)}
    # per-token int8 quantisation + INT8-MMA GEMM on a SYM blob of the 70B gate-up shape at
    # the headline width (the stack itself is W4A16; this is the variant's own kernel pair).
    a8 = None
    if args.lm_head and rank == 0 and world == 1:
        try:
            Ka, Na = dims.hidden, 2 * dims.ffn
            Wa = torch.empty(Ka, Na, dtype=torch.float16, device=dev)
            synth.gpu(args.seed, synth.tensor_id(0xFFC, 1, 0), synth.WEIGHT, Ka, Na, out=Wa)
            pla = w4.pack_linear(Wa, mode=w4.W4A16_SYM)
            del Wa
            Xa = synth.gpu(args.seed, synth.tensor_id(0xFFC, 2, 0), synth.ACT, M, Ka)
            Xqa = torch.empty(M, Ka, dtype=torch.int8, device=dev)
            sxa = torch.empty(M, dtype=torch.float32, device=dev)
            xsa = torch.empty(M, Ka // 128, dtype=torch.int32, device=dev)
            wsa8 = torch.zeros(w4.w4a8_workspace_bytes(M, Ka, Na), dtype=torch.uint8, device=dev)
            Ya = torch.empty(M, Na, dtype=torch.float16, device=dev)
            with torch.cuda.stream(stream):
                w4.w4a8_quantize_act(Xa, Xqa, sxa, xsa, stream=stream)
                w4.w4a8_gemm(Xqa, sxa, xsa, pla.packed, Ya, wsa8, stream=stream)
            torch.cuda.synchronize()
            g8a = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g8a, stream=stream):
                for _ in range(10):
                    w4.w4a8_quantize_act(Xa, Xqa, sxa, xsa, stream=stream)
                    w4.w4a8_gemm(Xqa, sxa, xsa, pla.packed, Ya, wsa8, stream=stream)
            ms8 = time_graph(g8a, 5, 2) / 10
            wb8 = Ka * Na // 2 + (Ka // 128) * Na * 2
            a8 = {"row": "f4", "shape": [M, Ka, Na], "mode": "SYM g128 weights, per-token int8 activations",
                  "us": 1e3 * ms8, "TBps": wb8 / (ms8 * 1e-3) / 1e12, "frac_hbm": wb8 / (ms8 * 1e-3) / 1e9 / peak_gbs,
                  "note": "quantise + GEMM per call; first version (DESIGN 5.10)"}
            log(f"W4A8 gate-up M={M}: {1e3 * ms8:.1f} us ({a8['TBps']:.2f} TB/s)")
            del g8a
        except Exception as e:   # never let the side measurement break the bench line
            a8 = {"row": "f4", "error": repr(e)}
    clk = clocks.stop() if clocks else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, sample, threads = oracle_layer_slice(M, args.seed)
        reps = max(1, min(50, int(6.0 / max(dt, 1e-3))))
        ts = [oracle_layer_slice(M, args.seed)[1] for _ in range(reps)]
        dt = statistics.median(ts)
        wb = sum(K * (N // 64) // 2 + (K // 128) * (N // 64) * 4 for K, N in SHAPES_70B.values())
        cpu = {"value": wb / dt / 1e12, "unit": "TB/s", "cores": threads, "kind": "oracle",
               "sample": sample + f", median of {reps} runs ({dt:.2f} s each)", "cpu_model": cpu_model()}
        log(f"cpu baseline (oracle, headline M): {cpu['value'] * 1e3:.3f} GB/s")
        try:
            cpu["plan"] = cpu_baseline_plan(M, args.seed)
            log("cpu baseline plan: " + json.dumps(cpu["plan"]))
        except Exception as e:   # never let the side measurement break the bench line
            cpu["plan"] = {"error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (seeded counter-based generator: N(0,0.018^2) weights with 2% x8 outlier groups, each "
                    "matrix scaled once by a power of two so its output RMS stays in [0.7, 1.4] along the data flow "
                    "(stand-in for the excluded norms); N(0,1.15^2) input activations with 4 x16 outlier channels; "
                    "EAGLE-2-shaped draft tree)",
            "config": {"workload": f"{dims.name} W4A16 g128 {args.mode} verify forward: {n_layers} decoder layers "
                                   f"(QKV -> O -> gate-up with SiLU*mul fused -> down -> next layer, each GEMM reading the "
                                   f"previous one's output; attention/norms out of scope) + verify_accept; "
                                   f"BASELINE configs 3-4",
                       "M": args.M, "layers": n_layers, "tp": world, "parallelism": f"tp{world}",
                       "allreduce": allreduce_used,
                       "weight_bytes_per_step": bytes_all_ranks,
                       "l2": f"{bytes_all_ranks / 1e9:.1f} GB of weights per step >> 126 MB L2 (no flush needed)",
                       "timing": f"CUDA graph replay, CUDA events on the launching stream, max over ranks; headline = median of "
                                 f"{args.windows} windows of {args.steps} steps"},
            "us_per_layer": 1e3 * ms / n_layers, "ms_per_step_distribution": step_dist,
            "frac_hbm": value * 1e3 / (peak_gbs * world),
            "m_sweep": m_sweep, "ratio_M64_over_M1": ratio_64, "hierarchical_us_per_token": hier,
            "m_sweep_sym": sym_sweep, "headline_windows_ms": windows_ms,
            "kernels": kernels, "roofline": roofline, "cpu_baseline": cpu, "lm_head_argmax": lm, "tree_attention": attn,
            "allreduce_in_chain": ar, "w4a8_gemm": a8,
            "other_configs": other_configs,
            "e2e": {"value": bytes_all_ranks / (ms_e2e * 1e-3) / 1e12, "unit": "TB/s", "ms_per_step": ms_e2e,
                    "h2d_bytes_per_step": stack.h2d_bytes(M), "d2h_bytes_per_step": stack.d2h_bytes(M),
                    "api": "VerifyStack.verify_host (pinned host buffers, graph replay, accept result read back)",
                    "accept_result": acc},
            "gpu_launches": stack.launches_per_forward(args.M) * args.steps,
            "clocks": clk, "build_s": build_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
