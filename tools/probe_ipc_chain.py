#!/usr/bin/env python
"""Two processes on ONE GPU running tensor-parallel chains with ALLREDUCE ops over CUDA-IPC regions
(PeerGroup.ipc): the kernels of the two contexts time-slice, so the flag protocol is exercised across
processes (slowly). Prints per-rank check results. Usage: python tools/probe_ipc_chain.py"""
import os, socket, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.multiprocessing as mp


def worker(rank, world, port, q):
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
    Y1, Y2 = torch.empty(M, H, dtype=torch.float16, device="cuda"), torch.empty(M, Kr, dtype=torch.float16, device="cuda")
    ch = w4.Chain([("gemm", X, pl, P1), ("allreduce", P1, Y1, g), ("gemm", Y1, pl2, P2), ("allreduce", P2, Y2, g)], M)
    ok = True
    times = []
    for rep in range(3):
        dist.barrier()
        t0 = time.time()
        ch()
        torch.cuda.synchronize()
        times.append(time.time() - t0)
        dist.barrier()   # both ranks done: the peers' partials are final
        for P, Y in ((P1, Y1), (P2, Y2)):
            off = P.data_ptr() - g.local.data_ptr()
            parts = [g.peer_region(p)[off: off + P.numel() * 2].view(torch.float16).float() for p in range(world)]
            want = (parts[0] + parts[1]).half()
            ok &= bool(torch.equal(want.view(torch.int16).view(-1), Y.view(torch.int16).view(-1)))
        dist.barrier()
    g.close()
    dist.destroy_process_group()
    q.put((rank, ok, [round(t, 4) for t in times]))


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps: p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps: p.join(timeout=60)
    print(sorted(res))
