"""C5 size sweep: forward complex128 FFT for n = 2^t, t = 4..30 on one GPU.

For every t: plan (default lifting), 3 warm-up executes, then back-to-back batches timed
with one CUDA event pair each (see run()): L2-hot, and L2-cold (1 GiB flush before every
execute, the flush-only batch subtracted).
Prints one JSON line per size and, with --md PATH, writes the markdown table.

    python tools/sweep.py --tmin 4 --tmax 30 --md profiles/r02_sweep.md [--oracle-tmax 26]

The oracle column comes from `bench.py --impl reference --t T` (the one place besides the
tests allowed to run oracle/), i.e. the Fig 3.9 / Fig 6.1 oracle on all host cores.
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


def _span(s, fn, reps):
    """seconds between two events around `reps` calls of fn on stream s."""
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) * 1e-3


def oracle_time(t):
    """seconds per oracle transform of 2^t on this host (bench.py's reference arm)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--t", str(t),
                        "--steps", "1" if t >= 25 else "3", "--warmup", "3"], capture_output=True, text=True,
                       timeout=3600)
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            d = json.loads(line)
            return d["ms_per_step"] * 1e-3, d["cpu_baseline"]["cores"]
    return None, None


def run(t, reps):
    """This box's CUDA event clock ticks in 2.048 us steps, so a transform of t <= 20 is
    not timed alone: 'hot' = one event pair around `reps` back-to-back executes, 'cold' =
    (reps x [1 GiB L2 flush + execute]) - (reps x flush), both / reps, median of 5.  From
    2^21 on: the median of `reps` executes each between its own event pair (after a flush
    for 'cold')."""
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

        def fft():
            plan.execute(x, out)

        def flush():
            fl.fill_(1.0)

        def both():
            fl.fill_(1.0)
            plan.execute(x, out)

        hot, cold = [], []
        if t <= 20:   # shorter than ~10 event ticks: batches
            for _ in range(5):
                hot.append(_span(s, fft, reps) / reps)
                cold.append((_span(s, both, reps) - _span(s, flush, reps)) / reps)
        else:         # one event pair per execute (tick <= 5 % of the transform)
            for _ in range(reps):
                flush()
                cold.append(_span(s, fft, 1))
            for _ in range(reps):
                hot.append(_span(s, fft, 1))
    info = plan.info()
    plan.destroy()
    cold.sort()
    hot.sort()
    tc, th = cold[len(cold) // 2], hot[len(hot) // 2]
    flops = 5.0 * n * t
    return {"t": t, "n": n, "lift": info["lift"], "passes": info["passes"], "launches": info["launches"],
            "us_cold": round(tc * 1e6, 2), "us_hot": round(th * 1e6, 2),
            "GFLOPs_cold": round(flops / tc / 1e9, 1), "GFLOPs_hot": round(flops / th / 1e9, 1),
            "alg_GBps_cold": round(info["hbm_bytes"] / tc / 1e9, 1), "hbm_bytes": info["hbm_bytes"],
            # 32 n ceil(t/13) bytes (the fewest <= 2^13-point passes)
            "survey_GBps_cold": round(32 * n * -(-t // 13) / tc / 1e9, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tmin", type=int, default=4)
    ap.add_argument("--tmax", type=int, default=30)
    ap.add_argument("--md", default="")
    ap.add_argument("--oracle-tmax", type=int, default=26)
    a = ap.parse_args()
    pk = peaks()
    rows = []
    for t in range(a.tmin, a.tmax + 1):
        reps = 20 if t <= 26 else 3
        r = run(t, reps)
        r["frac_of_measured_hbm"] = round(r["alg_GBps_cold"] / pk, 3)
        r["frac_survey"] = round(r["survey_GBps_cold"] / pk, 3)
        if t <= a.oracle_tmax:
            ot, cores = oracle_time(t)
            r["oracle_s"], r["oracle_cores"] = (round(ot, 6), cores) if ot is not None else (None, None)
        rows.append(r)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()
    if a.md:
        with open(a.md, "w") as f:
            f.write("# C5 size sweep, 1 B200, forward complex128 (default liftings)\n\n")
            f.write("Columns: plan bytes = 32 n x the plan's HBM passes ('alg GB/s', 'frac plan'); survey bytes = "
                    "32 n ceil(t/13), SURVEY §8(d) ('frac survey', the headline definition); oracle = the CPU "
                    "oracle (Fig 3.9, Fig 6.1 OpenMP mode on all host cores) per transform, via bench.py "
                    "--impl reference.\n\n")
            f.write(f"This box's CUDA event clock ticks in 2.048 us steps. t <= 20: 'hot' = one event pair "
                    f"around 20 back-to-back executes / 20; 'cold' = (20 x [1 GiB L2 flush + execute] minus "
                    f"20 x flush) / 20; median of 5 (for t <= ~15 'hot' is the CPU submission rate of "
                    f"back-to-back calls, 'cold' the GPU time). t >= 21: median of 20 (t <= 26) or 3 "
                    f"executes, each between its own event pair, after a flush for 'cold'. GFLOP/s = 5 n log2 n / t. alg GB/s = 32 n x HBM passes / t; fraction of "
                    f"the measured {pk} GB/s copy peak (MEASURED_PEAKS.json). Sizes <= 2^12 run in one CTA "
                    f"(latency-bound); up to ~2^22 the data is L2-resident between passes.\n\n")
            f.write("| t | lifting | launches | us (cold) | us (hot) | GFLOP/s (cold) | GFLOP/s (hot) | alg GB/s | "
                    "frac plan | frac survey | oracle s (cores) |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                orc = f"{r['oracle_s']} ({r['oracle_cores']})" if r.get("oracle_s") is not None else "-"
                f.write(f"| {r['t']} | {'x'.join(str(v) for v in r['lift'])} | {r['launches']} | {r['us_cold']} | "
                        f"{r['us_hot']} | {r['GFLOPs_cold']} | {r['GFLOPs_hot']} | {r['alg_GBps_cold']} | "
                        f"{r['frac_of_measured_hbm']} | {r['frac_survey']} | {orc} |\n")


if __name__ == "__main__":
    main()
