"""PCIe ceiling on this box (development tool): pinned H2D, D2H and both at once."""
import torch
n = 1 << 28  # 256 MiB
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3
def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
t1 = timed(h2d); t2 = timed(d2h); t3 = timed(both)
print(f"H2D {n/t1/1e9:.1f} GB/s  D2H {n/t2/1e9:.1f} GB/s  both: {2*n/t3/1e9:.1f} GB/s total ({n/t3/1e9:.1f} each)")
