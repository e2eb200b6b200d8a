"""Timing of the N2 layout redistributions on p virtual ranks of one B200 (dev tool).

On one GPU the transfers are device copies, so this measures the local side of each
route -- the pack / unpack kernels and the copy volume -- not NVLink.  Under torchrun
(one rank per GPU) the same plans run on real ranks over the library's NCCL
communicator: Fig 5.9's direct exchange against Fig 5.4's route through processor 0 on
NVSwitch, timed as the max over ranks.
python tools/redist_probe.py [t] [p]                       (p virtual ranks, one GPU)
torchrun --nproc-per-node P tools/redist_probe.py [t]      (P real ranks)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402

t = int(sys.argv[1]) if len(sys.argv) > 1 else 24
real = "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1
if real:
    import torch.distributed as dist
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl")
    moa.dist_init()
    p, rank = dist.get_world_size(), dist.get_rank()
else:
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rank = 0
n = 1 << t
B, C, Z = moa.LAYOUT_BLOCK, moa.LAYOUT_CYCLIC, moa.LAYOUT_CENTRAL
names = {B: "block", C: "cyclic", Z: "central"}
mode = moa.MODE_LIFTED if real else moa.MODE_EMULATED
for frm, to, route in [(B, C, 0), (B, C, 1), (C, B, 0), (C, B, 1), (Z, C, 0), (C, Z, 0), (Z, B, 0), (B, Z, 0)]:
    plan = moa.Redist(n, p, frm, to, route, mode=mode)
    cnt = plan.info()["elems_in"]
    x = torch.empty(max(cnt, 1), dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x08112535 + t, x.numel(), x)
    x = x if cnt else None
    out = plan.execute(x)
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(10):
        if real:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        plan.execute(x, out)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    med = ts[len(ts) // 2]
    if real:
        v = torch.tensor([med], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        med = float(v.item())
    info = plan.info()
    if rank == 0:
        print(json.dumps({"t": t, "p": p, "ranks": "real" if real else "virtual", "from": names[frm], "to": names[to],
                          "route": "central" if route else "direct", "us": round(med, 1),
                          "messages": info["messages"], "max_rank_bytes": info["max_rank_bytes"]}), flush=True)
    plan.destroy()

if real:
    moa.dist_finalize()
    dist.destroy_process_group()
