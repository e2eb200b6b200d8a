"""Dev check: the non-persistent TMA-loaded pass (MOA_FFT_TMA=3, variants library) against
cuFFT, then timings (run with MOA_BUILD_VARIANTS=1 MOA_FFT_ABLATION=1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402
from perf_probe import time_plan  # noqa: E402

print(moa.lib_path(), os.environ.get("MOA_FFT_TMA"))
for t, lift in [(24, None), (20, None), (22, None), (26, None), (16, None)]:
    n = 1 << t
    x = torch.empty(n, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x08112535 + t, n, x)
    plan = moa.Plan(n, lift=lift)
    plan.set_profiling(True)
    y = plan.execute(x)
    names = [k["name"] for k in plan.get_profile()]
    ref = torch.fft.fft(x)
    err = ((y - ref).abs().pow(2).sum() / ref.abs().pow(2).sum()).sqrt().item()
    print(t, f"relL2={err:.3e}", "OK" if err < 1e-12 * t else "FAIL", names, flush=True)
for t in (24, 26):
    print(time_plan(t, None), flush=True)
