"""Batched-transform throughput probe (development tool): GFLOP/s of `batch` x 2^t in one execute."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402

for spec in sys.argv[1:]:
    inplace = spec.endswith("i")
    t, batch = (int(v) for v in spec.rstrip("i").split("x"))
    n = 1 << t
    x = torch.empty(n * batch, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x1234 + t, n * batch, x)
    out = x if inplace else torch.empty_like(x)
    plan = moa.Plan(n, batch=batch)
    plan.set_profiling(True)
    for _ in range(3):
        plan.execute(x, out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record()
    for _ in range(reps):
        plan.execute(x, out)
    b.record()
    b.synchronize()
    dt = a.elapsed_time(b) * 1e-3 / reps
    info = plan.info()
    kern = [(k["name"][:26], round(k["avg_us"], 1)) for k in plan.get_profile()]
    print(json.dumps({"t": t, "batch": batch, "lift": info["lift"], "us": round(dt * 1e6, 1),
                      "GFLOPs": round(5 * n * t * batch / dt / 1e9, 1),
                      "alg_GBps": round(info["hbm_bytes"] / dt / 1e9, 1), "inplace": inplace,
                      "kernels": kern}), flush=True)
    del x, out, plan
