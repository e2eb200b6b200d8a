"""Small invocations of every kernel family, for compute-sanitizer (one tool per run):
    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
Checks results against torch.fft (cuFFT) so a sanitizer-clean run is also a correct one."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402


def check(got, ref, what):
    err = (torch.linalg.vector_norm(got - ref) / torch.linalg.vector_norm(ref)).item()
    assert err < 1e-12 * 32, (what, err)


def main():
    torch.manual_seed(0)
    for t, lift in [(4, None), (9, None), (13, None), (14, None), (16, [16, 16, 256]), (17, [32, 64, 64]),
                    (20, None), (21, None), (22, [16, 16, 64, 256])]:
        n = 1 << t
        x = torch.randn(n, dtype=torch.complex128, device="cuda")
        for sign in (-1, 1):
            got = moa.Plan(n, 1, sign, lift=lift).execute(x)
            ref = torch.fft.fft(x) if sign < 0 else torch.fft.ifft(x) * n
            check(got, ref, (t, lift, sign))
    x = torch.randn(8 * 1024, dtype=torch.complex128, device="cuda")
    check(moa.Plan(1024, batch=8).execute(x), torch.fft.fft(x.view(8, 1024)).reshape(-1), "batch")
    x = torch.randn(64, 512, dtype=torch.complex128, device="cuda")
    check(moa.Plan2D(64, 512).execute(x).view(64, 512), torch.fft.fft2(x), "2d")
    x = torch.randn(1 << 14, 4, dtype=torch.complex128, device="cuda")
    check(moa.PlanND((1 << 14, 4)).execute(x).view(1 << 14, 4), torch.fft.fft2(x), "nd-lifted")
    n, P = 1 << 12, 4
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    xin = torch.cat([x[r::P] for r in range(P)])
    ref = torch.fft.fft(x)
    for xchg in (moa.XCHG_NCCL, moa.XCHG_P2P):
        got = moa.Plan(n, P, -1, mode=moa.MODE_EMULATED, exchange=xchg).execute(xin).view(P, -1)
        for r in range(P):
            check(got[r], ref[r::P], ("emulated", xchg, r))
    got = moa.Plan(n, P, -1, mode=moa.MODE_EMULATED, breakpoint=3).execute(xin).view(P, -1)   # low end
    for r in range(P):
        check(got[r], ref[r::P], ("emulated low-end", r))
    for t in (9, 10):   # radix-2/4 remainder stages (xmask exchanges), row and column tiles
        m = 1 << t
        y = torch.randn(4 * m * m, dtype=torch.complex128, device="cuda")
        check(moa.Plan(m * m, lift=[m, m]).execute(y[:m * m]), torch.fft.fft(y[:m * m]), ("remainder", t))
        check(moa.Plan(m, batch=4 * m).execute(y), torch.fft.fft(y.view(4 * m, m)).reshape(-1), ("rem-batch", t))
    y = torch.randn(4096, 64, dtype=torch.complex128, device="cuda")
    check(moa.Plan2D(4096, 64).execute(y).view(4096, 64), torch.fft.fft2(y), "2d long column axis")
    got = moa.Plan(1 << 10, mode=moa.MODE_LITERAL).execute(x[:1024])
    check(got, torch.fft.fft(x[:1024]), "literal")
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
