"""One rank of the multi-GPU parity run (tests/test_gpu_multi.py launches it with
``python -m torch.distributed.run --nproc-per-node P tests/dist_worker.py T...``).

Each rank owns its own B200 (LOCAL_RANK), joins an NCCL process group and the
library's own NCCL communicator (moa.dist_init), generates its residue class
x[r + P j] of the seeded input and runs the partitioned transform with every
exchange the library has -- the NCCL send/recv group (Fig 5.9
P:1047-1062) unchunked and chunked (§8(e)), the fused NVLink push (MOA_XCHG_P2P,
§8(f) N1) and the low-end breakpoint -- then checks X[r + P i] element by
element against the CPU oracle's slice (relL2 <= 1e-12 log2 n), bitwise agreement
between the exchanges, and repeatability over three executes.  Rank 0 prints one
JSON line with every rank's errors and ``ALL-OK`` when everything passed.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import moa_inputs
    import oracle
    import paper_0811_2535_b200 as moa

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    moa.dist_init()
    ts = [int(v) for v in sys.argv[1:]] or [20]
    cores = max(1, len(os.sched_getaffinity(0)) // world)
    report, ok = [], True
    for t in ts:
        n = 1 << t
        M = n // world
        x = torch.empty(M, dtype=torch.complex128, device="cuda")
        moa.gen_uniform(moa_inputs.seed_for(t), M, x, first=rank, stride=world)
        ref = oracle.fft(moa_inputs.signal_for(t), -1, threads=cores)[rank::world]
        outs = {}
        cases = [("nccl", {}), ("nccl_unchunked", {"chunks": 1}), ("p2p", {"exchange": moa.XCHG_P2P})]
        if M >= 2 * world:
            cases.append(("low_end", {"breakpoint": world.bit_length()}))   # log2 p + 1
        for name, kw in cases:
            try:
                plan = moa.Plan(n, world, -1, **kw)
            except moa.MoaError as e:   # e.g. a two-level lifting has nothing to chunk
                report.append({"t": t, "case": name, "skipped": str(e)[:120]})
                continue
            if name == "p2p":
                plan.enable_p2p()
            runs = []
            for _ in range(3):
                runs.append(plan.execute(x).clone())
            torch.cuda.synchronize()
            same = all(torch.equal(runs[0], r) for r in runs[1:])
            err = oracle.rel_l2(runs[0].cpu().numpy(), ref)
            good = same and err <= 1e-12 * t
            ok &= good
            outs[name] = runs[0]
            report.append({"t": t, "case": name, "relL2": err, "repeatable": same, "info": plan.info()["chunks"]})
            plan.destroy()
        # the public one-call API, and the exchanges agree bit for bit (same arithmetic)
        y = moa.dist_fft(x, n)
        ok &= torch.equal(y, outs["nccl"]) and torch.equal(outs["p2p"], outs["nccl"])
        if "nccl_unchunked" in outs:
            ok &= torch.equal(outs["nccl_unchunked"], outs["nccl"])
        report.append({"t": t, "case": "bitwise nccl == p2p == dist_fft (== unchunked)", "ok": bool(ok)})
        # N2 on real ranks: the paper's layouts through the library (Fig 5.9 direct and Fig 5.4
        # through processor 0), bit-exact against numpy slices of the seeded input, and the
        # block-natural transform against the oracle's natural block
        xh = moa_inputs.signal_for(t)
        xb = torch.from_numpy(xh[rank * M:(rank + 1) * M].copy()).cuda()
        for route in (moa.ROUTE_DIRECT, moa.ROUTE_CENTRAL):
            c = moa.block_to_cyclic(xb, n, route)
            b = moa.cyclic_to_block(c, n, route)
            good = np.array_equal(c.cpu().numpy(), xh[rank::world]) and torch.equal(b, xb)
            ok &= good
            report.append({"t": t, "case": f"block<->cyclic route {route}", "ok": bool(good)})
        z = torch.from_numpy(xh).cuda() if rank == 0 else None
        c = moa.scatter_cyclic(z, n)
        g = moa.gather_cyclic(c, n)
        good = np.array_equal(c.cpu().numpy(), xh[rank::world]) and (rank != 0 or np.array_equal(g.cpu().numpy(), xh))
        ok &= good
        Xb = moa.dist_fft_block(xb, n)
        err = oracle.rel_l2(Xb.cpu().numpy(), oracle.fft(xh, -1, threads=cores)[rank * M:(rank + 1) * M])
        ok &= err <= 1e-12 * t
        report.append({"t": t, "case": "central scatter/gather, dist_fft_block", "ok": bool(good), "relL2": err})
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    reports = [None] * world
    dist.all_gather_object(reports, report)
    if rank == 0:
        print(json.dumps({"world": world, "ranks": reports}), flush=True)
        if int(flag.item()) == 1:
            print("ALL-OK", flush=True)
    moa.dist_finalize()
    dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) == 1 else 1)


if __name__ == "__main__":
    main()
