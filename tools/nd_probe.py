"""N3 throughput: batched 1-D, 2-D and 3-D transforms on one B200.

For each case: plan, 3 warm-up executes, then one CUDA event pair around REPS back-to-back
executes (inputs larger than L2 from 2^23 elements on); per-kernel times from a second,
profiled run.  GFLOP/s counts 5 N log2 N for the total size N of the transform (a batch of
b transforms of length n counts b * 5 n log2 n).  alg GB/s = 32 N x HBM passes / t.

    python tools/nd_probe.py --md profiles/r01_batched_nd.md
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402

CASES = [
    ("batch", (1 << 8, 1 << 16)), ("batch", (1 << 10, 1 << 14)), ("batch", (1 << 12, 1 << 12)),
    ("batch", (1 << 16, 1 << 8)), ("batch", (1 << 20, 1 << 4)),
    ("batch", (1 << 10, 1 << 16)), ("batch", (1 << 16, 1 << 10)),
    ("2d", (4096, 4096)), ("2d", (1024, 16384)), ("2d", (8192, 8192)),
    ("3d", (256, 256, 256)), ("3d", (512, 512, 256)),
]


def make(kind, dims):
    if kind == "batch":
        n, b = dims
        return moa.Plan(n, batch=b), n * b, b * 5.0 * n * math.log2(n)
    N = 1
    for d in dims:
        N *= d
    plan = moa.Plan2D(*dims) if kind == "2d" else moa.PlanND(dims)
    return plan, N, 5.0 * N * math.log2(N)


def run(kind, dims, reps=10):
    plan, N, flops = make(kind, dims)
    x = torch.empty(N, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x5EED + N, N, x)
    out = torch.empty_like(x)
    for _ in range(3):
        plan.execute(x, out)
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        plan.execute(x, out)
    b.record(s)
    b.synchronize()
    dt = a.elapsed_time(b) * 1e-3 / reps
    plan.set_profiling(True)
    plan.get_profile()
    for _ in range(reps):
        plan.execute(x, out)
    kern = [(k["name"], round(k["avg_us"], 1)) for k in plan.get_profile()]
    info = plan.info()
    plan.destroy()
    return {"kind": kind, "dims": list(dims), "N": N, "lift": info["lift"], "launches": info["launches"],
            "us": round(dt * 1e6, 1), "GFLOPs": round(flops / dt / 1e9, 1),
            "alg_GBps": round(info["hbm_bytes"] / dt / 1e9, 1), "kernels": kern}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--md", default="")
    a = ap.parse_args()
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except Exception:
        peak = 6650.0
    rows = []
    for kind, dims in CASES:
        r = run(kind, dims)
        r["frac"] = round(r["alg_GBps"] / peak, 3)
        rows.append(r)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()
    if a.md:
        with open(a.md, "w") as f:
            f.write("# N3: batched, 2-D and 3-D transforms (1 B200, forward complex128)\n\n"
                    "`python tools/nd_probe.py`: one event pair around 10 back-to-back executes; per-kernel "
                    "times from a second, profiled run. GFLOP/s = 5 N log2 N of the whole transform "
                    "(b x 5 n log2 n for a batch). alg GB/s = 32 N x HBM passes / t; frac = of the "
                    f"measured {peak} GB/s copy peak.\n\n"
                    "| kind | shape | lifting (1-D part) | launches | µs | GFLOP/s | alg GB/s | frac | kernels (µs) |\n"
                    "|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                shape = " x ".join(map(str, r["dims"])) if r["kind"] != "batch" else \
                    f"{r['dims'][1]} x 2^{int(math.log2(r['dims'][0]))}"
                ks = "; ".join(f"{k}: {v}" for k, v in r["kernels"])
                f.write(f"| {r['kind']} | {shape} | {'x'.join(map(str, r['lift']))} | {r['launches']} | {r['us']} | "
                        f"{r['GFLOPs']} | {r['alg_GBps']} | {r['frac']} | {ks} |\n")


if __name__ == "__main__":
    main()
