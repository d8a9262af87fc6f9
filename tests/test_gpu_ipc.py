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
