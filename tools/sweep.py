"""C5 size sweep: forward complex128 FFT for n = 2^t, t = 4..30 on one GPU.

For every t: plan (default lifting), 3 warm-up executes, then REPS executes timed one by
one with CUDA events on the plan stream, with a 1 GiB L2 flush before each (so
L2-resident sizes are reported L2-cold; the L2-hot median is reported beside it).
Prints one JSON line per size and, with --md PATH, writes the markdown table.

    python tools/sweep.py --tmin 4 --tmax 30 --md profiles/r01_sweep.md
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moa_inputs  # noqa: E402
import paper_0811_2535_b200 as moa  # noqa: E402


def peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def run(t, reps):
    n = 1 << t
    x = torch.empty(n, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(moa_inputs.seed_for(t), n, x)
    out = torch.empty_like(x)
    s = torch.cuda.Stream()
    plan = moa.Plan(n, stream=s)
    fl = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(3):
            plan.execute(x, out)
        cold, hot = [], []
        for flush, acc in ((True, cold), (False, hot)):
            for _ in range(reps):
                if flush:
                    fl.fill_(1.0)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(s)
                plan.execute(x, out)
                b.record(s)
                b.synchronize()
                acc.append(a.elapsed_time(b) * 1e-3)
    info = plan.info()
    plan.destroy()
    cold.sort()
    hot.sort()
    tc, th = cold[len(cold) // 2], hot[len(hot) // 2]
    flops = 5.0 * n * t
    return {"t": t, "n": n, "lift": info["lift"], "passes": info["passes"], "launches": info["launches"],
            "us_cold": round(tc * 1e6, 2), "us_hot": round(th * 1e6, 2),
            "GFLOPs_cold": round(flops / tc / 1e9, 1), "GFLOPs_hot": round(flops / th / 1e9, 1),
            "alg_GBps_cold": round(info["hbm_bytes"] / tc / 1e9, 1), "hbm_bytes": info["hbm_bytes"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tmin", type=int, default=4)
    ap.add_argument("--tmax", type=int, default=30)
    ap.add_argument("--md", default="")
    a = ap.parse_args()
    pk = peaks()
    rows = []
    for t in range(a.tmin, a.tmax + 1):
        reps = 20 if t <= 26 else 5
        r = run(t, reps)
        r["frac_of_measured_hbm"] = round(r["alg_GBps_cold"] / pk, 3)
        rows.append(r)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()
    if a.md:
        with open(a.md, "w") as f:
            f.write("# C5 size sweep, 1 B200, forward complex128 (default liftings)\n\n")
            f.write(f"Median of 20 (t <= 26) or 5 executes; L2 flushed (1 GiB write) before each 'cold' "
                    f"execute, none before 'hot'. GFLOP/s = 5 n log2 n / t. alg GB/s = 32 n x HBM passes / t; "
                    f"fraction of the measured {pk} GB/s copy peak (MEASURED_PEAKS.json). Sizes <= 2^13 run "
                    f"in one CTA (latency-bound); up to ~2^22 the data is L2-resident between passes. "
                    f"For launch-bound sizes the 'hot' column includes the CPU submission latency (the GPU "
                    f"is idle when the transform is launched), while in the 'cold' column the preceding flush "
                    f"kernel hides it.\n\n")
            f.write("| t | lifting | launches | us (cold) | us (hot) | GFLOP/s (cold) | GFLOP/s (hot) | alg GB/s | "
                    "frac HBM |\n|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['t']} | {'x'.join(str(v) for v in r['lift'])} | {r['launches']} | {r['us_cold']} | "
                        f"{r['us_hot']} | {r['GFLOPs_cold']} | {r['GFLOPs_hot']} | {r['alg_GBps_cold']} | "
                        f"{r['frac_of_measured_hbm']} |\n")


if __name__ == "__main__":
    main()
