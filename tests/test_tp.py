"""Tensor-parallel shard layer: host logic on CPU (-m "not gpu").

The shard plan (paper_2505_22179_b200/tp.py) is checked for coverage/alignment at t = 1, 2, 4, 8
for the Llama-3 8B/70B shapes, and the sharded computation is checked end to end with world_size 2 over gloo:
each rank quantises and multiplies ITS shard with the CPU oracle, row-parallel partials are summed with
all_reduce, column-parallel outputs are gathered, and the result must equal the oracle on the full matrices.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2505_22179_b200 import tp

TINY = tp.ModelDims("tiny", hidden=512, ffn=1024, n_q=4, n_kv=2, head=128, layers=2)


@pytest.mark.parametrize("dims", [tp.LLAMA3_8B, tp.LLAMA3_70B])
@pytest.mark.parametrize("t", [1, 2, 4, 8])
def test_shard_plan_partitions_every_matrix(dims, t):
    cover = {}
    for r in range(t):
        plan = tp.shard_plan(dims, t, r)
        for name, s in plan.items():
            K, N = s["full"]
            r0, r1 = s["rows"]
            assert s["K"] == r1 - r0 and s["N"] == sum(c1 - c0 for c0, c1 in s["cols"])
            assert s["K"] % 128 == 0 and s["N"] % 128 == 0            # packable, tile aligned
            assert all(c0 % 128 == 0 and c1 % 128 == 0 for c0, c1 in s["cols"]) and r0 % 128 == 0
            cells = cover.setdefault(name, np.zeros((K // 128, N // 128), dtype=np.int32))
            for c0, c1 in s["cols"]:
                cells[r0 // 128:r1 // 128, c0 // 128:c1 // 128] += 1
    for name, cells in cover.items():
        assert np.all(cells == 1), name                               # every 128x128 block exactly once


def test_shard_plan_head_alignment_70b_tp8():
    plan = tp.shard_plan(tp.LLAMA3_70B, 8, 3)
    assert plan["qkv"]["N"] == 1280 and plan["o"]["K"] == 1024          # 8 q heads + 1 kv head; its 8 q heads
    assert plan["gate_up"]["N"] == 7168 and plan["down"]["K"] == 3584
    assert plan["qkv"]["cols"][0] == (3 * 1024, 4 * 1024)                 # q heads 24..31
    assert plan["gate_up"]["cols"] == [(3 * 3584, 4 * 3584), (28672 + 3 * 3584, 28672 + 4 * 3584)]
    assert plan["down"]["rows"] == (3 * 3584, 4 * 3584)                   # matches the gate/up slice
    with pytest.raises(ValueError):
        tp.shard_plan(tp.LLAMA3_70B, 16, 0)                                # 8 kv heads cannot split 16 ways


def test_weight_bytes_partition():
    full = tp.weight_bytes(tp.LLAMA3_70B, 1)
    assert full == 80 * 454_557_696
    for t in (2, 4, 8):
        assert tp.weight_bytes(tp.LLAMA3_70B, t) * t == full


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tp_worker(rank, world, port, M, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = TINY
        errs = {}
        for li, name in enumerate(tp.MATRICES):
            spec = tp.shard_plan(d, world, rank)[name]
            K, N = spec["full"]
            W_full = torch.from_numpy(synth.host(5, synth.tensor_id(0, li), synth.WEIGHT, K, N).view(np.int16))
            X_full = synth.host(6, synth.tensor_id(0, li), synth.ACT, M, K)
            W_r = tp.shard_of(W_full, spec).numpy().view(np.uint16)
            r0, r1 = spec["rows"]
            X_r = np.ascontiguousarray(X_full[:, r0:r1])
            codes, sc, ze, _ = oracle.quantize(W_r)
            Y_r = torch.from_numpy(oracle.gemm(X_r, codes, sc, ze))
            if name in ("o", "down"):                      # row-parallel: partial sums, all-reduce
                dist.all_reduce(Y_r)
                Y = Y_r.numpy()
            else:                                          # column-parallel: gather the column shards
                parts = [torch.zeros_like(Y_r) for _ in range(world)]
                dist.all_gather(parts, Y_r)
                Y = np.zeros((M, N))
                for rr in range(world):
                    off = 0
                    for c0, c1 in tp.shard_plan(d, world, rr)[name]["cols"]:
                        Y[:, c0:c1] = parts[rr].numpy()[:, off:off + c1 - c0]
                        off += c1 - c0
            if rank == 0:
                c_full, s_full, z_full, _ = oracle.quantize(W_full.numpy().view(np.uint16))
                ref = oracle.gemm(X_full, c_full, s_full, z_full, nthreads=2)
                errs[name] = float(np.abs(Y - ref).max() / (1 + np.abs(ref).max()))
        if rank == 0:
            result_q.put(errs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M", [3, 16])
def test_sharded_verify_layer_equals_full_oracle_gloo(M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, M, q)) for r in range(2)]
    for p in procs:
        p.start()
    errs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # column shards reproduce the full result exactly (same per-column arithmetic); row shards differ only by
    # the fp64 summation order of the all-reduce
    assert errs["qkv"] == 0.0 and errs["gate_up"] == 0.0
    assert errs["o"] < 1e-12 and errs["down"] < 1e-12
