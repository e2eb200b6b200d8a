"""Lifting / tile-size tuning probe for the mid sizes (development tool, not the bench).

For every t, every candidate lifting and every (MOA_FFT_MINTILES, MOA_FFT_TF) setting:
median of REPS L2-flushed executes (tools/perf_probe.time_plan).  The env knobs are read at
plan creation, so they are set in-process between plans.

    python tools/tune_probe.py 17 23 > gpurun_out/tune.jsonl
    python tools/tune_probe.py 25 28 big > gpurun_out/tune_big.jsonl
"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import perf_probe  # noqa: E402


def time_batched(t, lift, reps=20):
    """L2-cold time of one execute below the 2.048 us event tick: (reps x [1 GiB flush +
    execute] - reps x flush) / reps, median of 3 (tools/sweep.py's method)."""
    import torch
    import paper_0811_2535_b200 as moa
    n = 1 << t
    x = torch.empty(n, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x08112535 + t, n, x)
    out = torch.empty_like(x)
    plan = moa.Plan(n, lift=lift)
    fl = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()

    def span(fn):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        b.synchronize()
        return a.elapsed_time(b) * 1e-3

    for _ in range(3):
        plan.execute(x, out)
    ts = []
    for _ in range(3):
        both = span(lambda: (fl.fill_(1.0), plan.execute(x, out)))
        only = span(lambda: fl.fill_(1.0))
        ts.append((both - only) / reps)
    ts.sort()
    info = plan.info()
    plan.destroy()
    return {"t": t, "lift": info["lift"], "us": round(ts[1] * 1e6, 2), "us_min": round(ts[0] * 1e6, 2),
            "tf": os.environ.get("MOA_FFT_TF", "default"), "kernels": []}


def liftings(t):
    out = []
    for a in range(max(1, t - 13), min(13, t - 1) + 1):
        out.append([1 << a, 1 << (t - a)])
    for a in range(3, 9):
        for b in range(5, 11):
            c = t - a - b
            if 5 <= c <= 12:
                out.append([1 << a, 1 << b, 1 << c])
    return out


def liftings_big(t):
    """3-level liftings with factors in [2^5, 2^12] and 4-level ones in [2^4, 2^10]."""
    out = []
    for a in range(5, 13):
        for b in range(5, 13):
            c = t - a - b
            if 5 <= c <= 12:
                out.append([1 << a, 1 << b, 1 << c])
    for a in range(4, 11):
        for b in range(4, 11):
            for c in range(4, 11):
                e = t - a - b - c
                if 4 <= e <= 10:
                    out.append([1 << a, 1 << b, 1 << c, 1 << e])
    return out


def main():
    t0, t1 = int(sys.argv[1]), int(sys.argv[2])
    big = len(sys.argv) > 3 and sys.argv[3] == "big"   # default knobs, 3 reps, 3/4-level liftings
    for t in range(t0, t1 + 1):
        best = None
        for lift in (liftings_big(t) if big else liftings(t)):
            for mt, tf in (((128, 8192),) if big else itertools.product((128, 296, 592), (2048, 4096, 8192))):
                if not big:   # big: the plan's own T rules
                    os.environ["MOA_FFT_MINTILES"] = str(mt)
                    os.environ["MOA_FFT_TF"] = str(tf)
                try:
                    r = (perf_probe.time_plan(t, lift, reps=3) if big else time_batched(t, lift))
                except Exception as e:   # unsupported (F, T) combination
                    print(json.dumps({"t": t, "lift": lift, "mintiles": mt, "tf": tf, "error": str(e)[:80]}))
                    continue
                r["mintiles"] = mt
                print(json.dumps(r), flush=True)
                if best is None or r["us"] < best["us"]:
                    best = r
        os.environ.pop("MOA_FFT_MINTILES", None)
        os.environ.pop("MOA_FFT_TF", None)
        d = perf_probe.time_plan(t, None, reps=3) if big else time_batched(t, None)
        print(json.dumps({"t": t, "default": d["lift"], "default_us": d["us"], "best": best["lift"],
                          "best_us": best["us"], "best_mintiles": best["mintiles"], "best_tf": best["tf"]}),
              flush=True)


if __name__ == "__main__":
    main()
