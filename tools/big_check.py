"""Dev check of the persistent 4096-point pass (bigpass.cu): results against torch.fft
(cuFFT) for liftings that use it, then timings against the default lifting."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402
from perf_probe import time_plan  # noqa: E402

cases = [(24, [4096, 4096]), (20, [256, 4096]), (20, [4096, 256]), (23, [2048, 4096]), (23, [4096, 2048]),
         (26, [16, 4096, 1024]), (26, [4, 4096, 4096]), (25, [4096, 8192]), (13, [2, 4096])]
for t, lift in cases:
    n = 1 << t
    x = torch.empty(n, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x08112535 + t, n, x)
    for sign in (-1, 1):
        plan = moa.Plan(n, 1, sign, lift=lift)
        plan.set_profiling(True)
        y = plan.execute(x)
        names = [k["name"] for k in plan.get_profile()]
        ref = torch.fft.fft(x) if sign < 0 else torch.fft.ifft(x) * n
        err = ((y - ref).abs().pow(2).sum() / ref.abs().pow(2).sum()).sqrt().item()
        print(t, lift, sign, f"relL2={err:.3e}", "OK" if err < 1e-12 * t else "FAIL", names, flush=True)
        plan.destroy()
for t, lift in [(24, None), (24, [4096, 4096]), (23, [2048, 4096]), (26, [4, 4096, 4096]), (28, [16, 4096, 4096])]:
    print(time_plan(t, lift), flush=True)
