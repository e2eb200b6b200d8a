"""Per-rank kernel time of a p > 1 plan for explicit local liftings, on p virtual ranks of
one B200 (dev tool): python tools/lift_p_probe.py T P LIFT [LIFT ...]   (LIFT = "a,b,c", "" = default)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402

t, P = int(sys.argv[1]), int(sys.argv[2])
n = 1 << t
x = torch.empty(n, dtype=torch.complex128, device="cuda")
moa.gen_uniform(0x08112535 + t, n, x)
out = torch.empty_like(x)
for spec in sys.argv[3:] or [""]:
    lift = [int(v) for v in spec.split(",")] if spec else None
    plan = moa.Plan(n, P, -1, mode=moa.MODE_EMULATED, lift=lift, exchange=moa.XCHG_P2P)
    for _ in range(2):
        plan.execute(x, out)
    plan.set_profiling(True)
    plan.get_profile()
    for _ in range(3):
        plan.execute(x, out)
    prof = plan.get_profile()
    per_rank = {k["name"]: round(k["avg_us"], 1) for k in prof}
    print(json.dumps({"t": t, "P": P, "lift": plan.info()["lift"], "per_rank_us": round(sum(per_rank.values()), 1),
                      "kernels": per_rank}), flush=True)
    plan.destroy()
    torch.cuda.empty_cache()
