"""CUDA-IPC symmetric regions (include/w4a16.h w4a16_ipc_*; ops.PeerGroup.ipc): two processes on one GPU
(gloo rendezvous on 127.0.0.1) allocate their regions, exchange handles, map each other's region and read
what the peer wrote; the carve-out offsets agree across ranks. The one-GPU box cannot run two chains of
different processes concurrently, so the in-kernel protocol itself is covered by test_gpu_allreduce.py
(simulated ranks in one process)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        import paper_2505_22179_b200 as w4
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        g = w4.PeerGroup.ipc(1 << 20, 4)
        a, b = g.alloc(16, 1024), g.alloc(8, 256)
        offs = (a.data_ptr() - g.local.data_ptr(), b.data_ptr() - g.local.data_ptr())
        a.fill_(float(rank + 1))
        torch.cuda.synchronize()
        dist.barrier()
        ok = True
        for p in range(world):
            reg = g.peer_region(p)
            view = reg[offs[0]: offs[0] + a.numel() * 2].view(torch.float16)
            ok &= bool(torch.all(view == float(p + 1)).item())
            ok &= bool(torch.all(reg[:w4.w4a16_peer_flag_bytes(4)] == 0).item())   # flag area zero-filled
        dist.barrier()
        g.close()
        dist.destroy_process_group()
        q.put((rank, ok, offs))
    except Exception as e:   # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.timeout(300)
def test_ipc_regions_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert res[0][2] == res[1][2]   # symmetric offsets


def _chain_worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        import paper_2505_22179_b200 as w4
        import synth
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        M, Kr, H = 8, 2048, 1280
        g = w4.PeerGroup.ipc(1 << 22, 4)
        pl = w4.pack_linear(synth.gpu(5, 100 + rank, synth.WEIGHT, Kr, H))
        pl2 = w4.pack_linear(synth.gpu(5, 200 + rank, synth.WEIGHT, H, Kr))
        X = synth.gpu(5, 300 + rank, synth.ACT, M, Kr)
        P1, P2 = g.alloc(M, H), g.alloc(M, Kr)
        Y1 = torch.empty(M, H, dtype=torch.float16, device="cuda")
        Y2 = torch.empty(M, Kr, dtype=torch.float16, device="cuda")
        ch = w4.Chain([("gemm", X, pl, P1), ("allreduce", P1, Y1, g), ("gemm", Y1, pl2, P2), ("allreduce", P2, Y2, g)], M)
        ok = True
        for rep in range(3):
            dist.barrier()
            ch()
            torch.cuda.synchronize()
            dist.barrier()   # every rank's partials are final
            for P, Y in ((P1, Y1), (P2, Y2)):
                off = P.data_ptr() - g.local.data_ptr()
                parts = [g.peer_region(p)[off: off + P.numel() * 2].view(torch.float16).float() for p in range(world)]
                want = (parts[0] + parts[1]).half()   # two fp16 terms: the fp32 sum rounded once
                ok &= bool(torch.equal(want.view(torch.int16).view(-1), Y.view(torch.int16).view(-1)))
            dist.barrier()
        dist.barrier()
        g.close()
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception as e:   # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.timeout(300)
def test_allreduce_chain_across_two_processes():
    """The real multi-process path (CUDA IPC regions, flags through peer mappings, one cooperative chain per
    process). On one GPU the two contexts' kernels time-slice, so each run takes milliseconds, but the
    protocol is the one NVLink peers use: every rank must end with the same rank-order sum of both partials."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
