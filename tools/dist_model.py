"""Per-rank phase costs of the partitioned transform, measured on ONE B200 as p virtual
ranks (MOA_MODE_EMULATED: the same per-rank kernels), plus a MODELLED exchange time.

Every gpurun call gets one GPU, so the p > 1 path cannot be timed end to end here.  This
tool times what each rank's GPU would run -- the local lifted passes of its n/p-point
FFT (the last one packing / pushing), and pcombine -- and adds the all-to-all as
bytes / link bandwidth (770 GB/s per direction: the measured NVLink peer copy in
B200_PROFILING.md).  The modelled line is labelled as such; it is not a measurement.

    python tools/dist_model.py --t 24 --md profiles/r01_dist_model.md
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_2535_b200 as moa  # noqa: E402

LINK_GBPS = 770.0


def measure(t, P, exchange, reps=10, breakpoint=0):
    n = 1 << t
    x = torch.empty(n, dtype=torch.complex128, device="cuda")
    moa.gen_uniform(0x08112535 + t, n, x)
    out = torch.empty_like(x)
    plan = moa.Plan(n, P, -1, mode=moa.MODE_EMULATED, exchange=exchange, breakpoint=breakpoint)
    for _ in range(3):
        plan.execute(x, out)
    torch.cuda.synchronize()
    plan.set_profiling(True)
    plan.get_profile()
    for _ in range(reps):
        plan.execute(x, out)
    prof = plan.get_profile()
    plan.set_profiling(False)
    info = plan.info()
    plan.destroy()
    # slots aggregate the p virtual ranks' launches: per-rank time = total / (reps * P)
    per_rank = {k["name"]: k["avg_us"] * k["launches"] / (reps * P) for k in prof}
    return per_rank, info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, nargs="+", default=[24])
    ap.add_argument("--md", default="")
    a = ap.parse_args()
    rows = []
    for t in a.t:
        n = 1 << t
        for P in (2, 4, 8):
            for xname, xchg, bp in (("nccl", moa.XCHG_NCCL, 0), ("p2p", moa.XCHG_P2P, 0),
                                    ("nccl, low-end breakpoint", moa.XCHG_NCCL, P.bit_length())):
                per_rank, info = measure(t, P, xchg, breakpoint=bp)
                M = n // P
                a2a_bytes = 16 * M * (P - 1) // P
                compute = sum(v for k, v in per_rank.items())
                t_a2a = a2a_bytes / (LINK_GBPS * 1e9) * 1e6
                # NCCL: compute, then the exchange, then pcombine (no overlap);
                # P2P: the exchange is stores of the last pass -> the last pass is bounded
                # below by its NVLink bytes (overlap inside the kernel)
                if xname.startswith("nccl"):
                    model = compute + t_a2a
                else:
                    last = max((v for k, v in per_rank.items() if k.startswith("pass")), default=0.0)
                    model = compute - last + max(last, t_a2a)
                r = {"t": t, "P": P, "exchange": xname, "lift": info["lift"], "breakpoint": info["breakpoint"],
                     "per_rank_kernels_us": {k: round(v, 1) for k, v in per_rank.items()},
                     "per_rank_compute_us": round(compute, 1), "a2a_bytes_per_rank": a2a_bytes,
                     "a2a_us_model_at_770GBps": round(t_a2a, 1), "per_gpu_us_model": round(model, 1),
                     "GFLOPs_model": round(5 * n * t / (model * 1e-6) / 1e9, 1)}
                rows.append(r)
                print(json.dumps(r), flush=True)
    if a.md:
        with open(a.md, "w") as f:
            f.write("# Partitioned transform: measured per-rank kernels + MODELLED exchange\n\n"
                    "One B200, p virtual ranks (`MOA_MODE_EMULATED`, the per-rank kernels of the real "
                    "p-GPU path). Per-rank kernel times are measured (CUDA events, per-rank share of the "
                    "emulated launches); the all-to-all is MODELLED as bytes / 770 GB/s (measured NVLink "
                    "peer copy, B200_PROFILING.md). NCCL: compute + exchange, no overlap. P2P: the last "
                    "pass stores into the peers, so it is bounded below by its NVLink bytes. These are "
                    "projections, not multi-GPU measurements. The low-end breakpoint (SURVEY N4, P:694) "
                    "runs psplit (the first log2 p stages + weightcyclic) before the exchange and the "
                    "whole local FFT after it.\n\n")
            f.write("| n | p | exchange | lifting (n/p) | per-rank kernels (µs) | exchange B/rank | "
                    "exchange µs (model) | per-GPU µs (model) | GFLOP/s (model) |\n"
                    "|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                ks = "; ".join(f"{k}: {v}" for k, v in r["per_rank_kernels_us"].items())
                f.write(f"| 2^{r['t']} | {r['P']} | {r['exchange']} | {'x'.join(map(str, r['lift']))} | {ks} | "
                        f"{r['a2a_bytes_per_rank']} | {r['a2a_us_model_at_770GBps']} | {r['per_gpu_us_model']} | "
                        f"{r['GFLOPs_model']} |\n")
            f.write("\n## N2: Fig 5.9 direct vs Fig 5.4 via-central redistribution (MODEL)\n\n"
                    "Bytes / 770 GB/s per link direction. Direct (Fig 5.9, P:1043): every rank sends "
                    "(m-1)/m of its psize elements to the others at once. Via central (Fig 5.4, P:844): "
                    "processor 0 receives (m-1) blocks of psize and sends (m-1) cyclic slices of psize "
                    "through its own link: 2(m-1) messages, every element moved twice, rank 0's link "
                    "the bottleneck (its two directions overlap: max of in and out).\n\n"
                    "| n | p | direct µs | via central µs | ratio |\n|---|---|---|---|---|\n")
            for t in a.t:
                n = 1 << t
                for P in (2, 4, 8):
                    M = n // P
                    direct = 16 * M * (P - 1) / P / (LINK_GBPS * 1e9) * 1e6
                    central = 16 * M * (P - 1) / (LINK_GBPS * 1e9) * 1e6   # rank 0: (m-1) psize each way
                    f.write(f"| 2^{t} | {P} | {direct:.1f} | {central:.1f} | {central / direct:.1f}x |\n")


if __name__ == "__main__":
    main()
