"""World-size-2 gloo tests of the multi-process host path (CPU, no GPU).

* the NCCL unique id made by the library on rank 0 reaches rank 1 intact through
  torch.distributed (the rendezvous dist_init uses);
* the partitioned plan's host maps (moa_fft_describe_pass: local lifted passes,
  rank twiddle omega_n^(r*K), pack to [dst][K/p]) driven through a REAL two-process
  exchange (gloo all_to_all_single, the S7 step) and the P-point combine give each
  rank X[r + p*i] of the oracle;
* bench.py --impl reference under torchrun: rank 0 prints the JSON line, rank 1 exits 0.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, t, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import moa_inputs
        import oracle
        import paper_0811_2535_b200 as moa
        from test_plan_maps import pcombine, replay_local

        ident = moa.bcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, ident)
        same_id = all(i == ids[0] for i in ids) and len(ident) == 128 and any(ident)

        n = 1 << t
        p = world
        m = n // p
        chunk = m // p
        x_local = moa_inputs.rank_slice(t, rank, p)
        send = replay_local(x_local, n, p, rank)                 # S5 + S6 from the product's maps
        recv = torch.empty(2 * m, dtype=torch.float64)
        dist.all_to_all_single(recv, torch.from_numpy(send.view(np.float64).copy()),
                               [2 * chunk] * p, [2 * chunk] * p)  # S7 over a real process boundary
        out = pcombine(recv.numpy().view(np.complex128), p)        # S8
        ref = oracle.fft(moa_inputs.signal_for(t), -1)[rank::p]
        err = oracle.rel_l2(out, ref)
        q.put((rank, same_id, err))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("t", [10, 16])
def test_two_rank_exchange_over_gloo(t):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, t, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, same_id, err in res:
        assert not isinstance(err, str), err
        assert same_id, "unique id differs across ranks"
        assert err <= 1e-13, (rank, err)


def test_bench_reference_arm_torchrun_two_ranks():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "3", "--t", "12"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["value"] > 0
    assert rec["cpu_baseline"]["kind"] == "oracle"
    assert rec["e2e"]["h2d_bytes_per_step"] == 0


def _layout_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import moa_inputs
        import paper_0811_2535_b200 as moa
        n = 1 << 10
        x0 = torch.from_numpy(moa_inputs.signal_for(10)) if rank == 0 else None
        import _layouts_torch as lt
        mine = lt.scatter_cyclic(x0, n)
        ok_scatter = np.array_equal(mine.numpy(), moa_inputs.signal_for(10)[rank::world])
        back = lt.gather_cyclic(mine, n)
        ok_gather = (rank != 0) or np.array_equal(back.numpy(), moa_inputs.signal_for(10))
        q.put((rank, bool(ok_scatter and ok_gather)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_centralized_cyclic_layouts_over_gloo(world):
    """Fig 5.8's centralized<->cyclic redistributions (scatter_cyclic /
    gather_cyclic): rank r gets x[r::p]; gathering the cyclic slices restores x."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_layout_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] is True for r in range(world)), res


def _block_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import moa_inputs
        import oracle
        import paper_0811_2535_b200 as moa
        from test_plan_maps import pcombine, replay_local
        t = 12
        n = 1 << t
        p = world
        m = n // p
        chunk = m // p
        x = moa_inputs.signal_for(t)
        xb = torch.from_numpy(x[rank * m:(rank + 1) * m].copy())
        import _layouts_torch as lt
        xc = lt.block_to_cyclic(xb)                                      # Fig 5.3 / 5.9 direct
        ok_direct = np.array_equal(xc.numpy(), x[rank::p])
        xv = lt.block_to_cyclic_via_central(xb)                          # Fig 5.4 via processor 0
        ok_central = np.array_equal(xv.numpy(), x[rank::p])
        # the partitioned transform on the cyclic slice (product maps + a real exchange),
        # then the output back to natural blocks: X[r*psize : (r+1)*psize]
        send = replay_local(xc.numpy(), n, p, rank)
        recv = torch.empty(2 * m, dtype=torch.float64)
        dist.all_to_all_single(recv, torch.from_numpy(send.view(np.float64).copy()),
                               [2 * chunk] * p, [2 * chunk] * p)
        Xc = torch.from_numpy(pcombine(recv.numpy().view(np.complex128), p).copy())
        Xb = lt.cyclic_to_block(Xc)
        ref = oracle.fft(x, -1)
        err = oracle.rel_l2(Xb.numpy(), ref[rank * m:(rank + 1) * m])
        q.put((rank, (ok_direct, ok_central, err)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_block_natural_layouts_over_gloo(world):
    """block-natural input and output around the cyclic transform
    (block_to_cyclic, cyclic_to_block: one all-to-all each) and Fig 5.4's via-central
    redistribution (gather to processor 0, scatter back: 2(m-1) messages) -- both give
    rank r exactly x[r::p]; the natural blocks of the result equal the oracle's X."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_block_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        ok_direct, ok_central, err = res[r]
        assert ok_direct and ok_central, (r, res[r])
        assert err <= 1e-13, (r, err)

