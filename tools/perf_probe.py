"""Quick timing probe of moa plans (development tool, not the bench).

python tools/perf_probe.py 24 "4096,4096" "2048,8192" ...   (env MOA_FFT_TF caps T*F)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402


def time_plan(t, lift, reps=10, mode=moa.MODE_LIFTED, flush=True):
    n = 1 << t
    x = torch.empty(n, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x08112535 + t, n, x)
    out = torch.empty_like(x)
    plan = moa.Plan(n, lift=lift, mode=mode)
    s = torch.cuda.current_stream()
    fl = torch.empty(1 << 28, dtype=torch.float32, device="cuda")   # 1 GiB > L2
    for _ in range(3):
        plan.execute(x, out)
    ts = []
    for _ in range(reps):
        if flush:
            fl.fill_(1.0)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        plan.execute(x, out)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    tmed = ts[len(ts) // 2]
    plan.set_profiling(True)
    plan.get_profile()
    for _ in range(reps):
        if flush:
            fl.fill_(1.0)
        plan.execute(x, out)
    kern = [(k["name"], round(k["avg_us"], 1), round(k["alg_bytes"] / k["avg_us"] / 1e3, 1))
            for k in plan.get_profile()]
    plan.set_profiling(False)
    info = plan.info()
    gbs = info["hbm_bytes"] / tmed / 1e9
    gf = 5 * n * t / tmed / 1e9
    return {"t": t, "lift": info["lift"], "mode": mode, "us": round(tmed * 1e6, 1),
            "us_min": round(ts[0] * 1e6, 1), "alg_GBps": round(gbs, 1), "GFLOPs": round(gf, 1),
            "tf": os.environ.get("MOA_FFT_TF", "8192"), "kernels": kern}


def calibrate():
    """copy bandwidth (read+write bytes) of a 1 GiB tensor and the SM clock: box sanity check."""
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    clk = None
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        pass
    del a, b
    return {"copy_GBps": round(2 * (1 << 30) / min(ts) / 1e9, 1), "sm_mhz": clk}


if __name__ == "__main__":
    print(json.dumps({"calibration": calibrate()}), flush=True)
    t = int(sys.argv[1])
    for spec in sys.argv[2:] or [""]:
        if spec == "literal":
            r = time_plan(t, None, mode=moa.MODE_LITERAL, reps=3)
        else:
            lift = [int(v) for v in spec.split(",")] if spec else None
            r = time_plan(t, lift)
        print(json.dumps(r), flush=True)
