"""The fused P2P exchange across a real process boundary (GPU box, one B200).

Two or four processes (gloo rendezvous on 127.0.0.1) each own a
MOA_XCHG_P2P_EXTERNAL plan on cuda:0.  They swap the CUDA-IPC handles of their
receive buffers through torch.distributed, so each process's last butterfly
pass stores (p-1)/p of its output straight into the OTHER processes' buffers (the
Fig 5.9 redistribution, fused into the kernel).  Between phase 1
and phase 2 the ranks meet at a host barrier (stream synchronise + gloo), so no
kernel ever waits on another process's kernel.  Each rank must end with
X[r + p i] of the oracle (xcyclic), over several executes (the
double-buffered receive halves alternate).
"""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, t, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import moa_inputs
        import oracle
        import paper_0811_2535_b200 as moa

        n = 1 << t
        m = n // world
        plan = moa.Plan(n, world, -1, exchange=moa.XCHG_P2P_EXTERNAL, rank=rank)
        plan.enable_p2p()
        x = torch.empty(m, dtype=torch.complex128, device="cuda")
        moa.gen_uniform(moa_inputs.seed_for(t), m, x, first=rank, stride=world)
        out = torch.empty_like(x)
        ref = oracle.fft(moa_inputs.signal_for(t), -1, threads=4)[rank::world]
        errs = []
        for _ in range(3):
            out.zero_()
            plan.execute_phase(x, None, 1)
            torch.cuda.synchronize()
            dist.barrier()
            plan.execute_phase(None, out, 2)
            torch.cuda.synchronize()
            dist.barrier()
            errs.append(oracle.rel_l2(out.cpu().numpy(), ref))
        plan.destroy()
        q.put((rank, max(errs)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("t,world", [(12, 2), (20, 2), (21, 4), (24, 4)])
def test_p2p_exchange_processes_one_gpu(t, world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, t, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        assert res[r] <= 1e-12 * t, (r, res[r])
