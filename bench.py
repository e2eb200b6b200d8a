#!/usr/bin/env python
"""Benchmark of the MoA reshape-transpose FFT on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--t 24]

A step is one complete forward complex128 FFT of n = 2^t (default t = 24,
BASELINE.json configs[2], the size the metric's >= 60 % HBM target is quoted
on), inputs resident in HBM, through the C ABI (moa_fft_execute).  With N > 1
(torchrun, one rank per GPU, NCCL) the same transform is partitioned p = N
ways (reshape-transpose with one all-to-all): strong scaling.

metric  = GFLOP/s counted as 5 n log2 n per transform (BASELINE.json metric)
roofline= the dominant kernel's algorithmic bytes / its event-timed launch
          duration against MEASURED_PEAKS.json hbm_gbs
e2e     = same metric through moa_fft_execute_host_batch (pinned host in/out,
          every step's H2D + transform + D2H inside the timed region; the copies
          of neighbouring steps overlap the transform on PCIe's two directions)
cpu_baseline / --impl reference = the CPU oracle (oracle/, Fig 3.9 + Fig 6.1
          OpenMP mode) timed on this host's cores -- a baseline, not the target.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "complex128 1-D FFT GFLOP/s (5n log2 n) and HBM GB/s fraction, 1/2/4/8 B200"
UNIT = "GFLOP/s"
L2_BYTES = 126 * 1000 * 1000   # B200 L2 (B200_PROFILING.md)


def flops(n: int) -> float:
    return 5.0 * n * (n.bit_length() - 1)


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(kernel_name: str, n: int, p: int):
    """dram bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{kernel_name}|n={n}|p={p}")
    except Exception:
        return None


class ClockSampler:
    """NVML polling of SM clock + throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting", 0x10: "sync_boost", 0x100: "display_clock_setting"}

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - NVML missing
            self.err = str(e)

    def _sample(self):
        nv = self._nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for bit, name in self.REASONS.items():
            if r & bit and name != "gpu_idle":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._h is not None:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- CPU oracle
def cpu_oracle_rate(t: int, reps: int):
    """The oracle as it stands (Fig 3.9; Fig 6.1 parallel-do mode on all host cores)."""
    import moa_inputs
    import oracle
    cores = len(os.sched_getaffinity(0))
    x = moa_inputs.signal_for(t)
    oracle.fft(x[:1 << 10], -1, threads=cores)  # load + build
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.fft(x, -1, threads=cores)
    dt = (time.perf_counter() - t0) / reps
    return flops(1 << t) / dt / 1e9, cores, dt


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, rank: int, world: int):
    """--impl reference: the CPU oracle on this host, same config/metric (rank 0 only)."""
    if rank != 0:
        return
    import moa_inputs
    import oracle
    t = args.t
    n = 1 << t
    cores = len(os.sched_getaffinity(0))
    x = moa_inputs.signal_for(t)
    for _ in range(args.warmup):
        oracle.fft(x, -1, threads=cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.fft(x, -1, threads=cores)
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    value = args.steps * flops(n) / total / 1e9
    sample = f"each step = one full n=2^{t} oracle transform (Fig 3.9 radix-2, Fig 6.1 OpenMP mode)"
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(t, world, None, l2_flush=16 * (n // world) < 2 * L2_BYTES),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu": cpu_model()},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(t: int, world: int, info, exchange: str = "nccl", l2_flush: bool = False):
    c = {"workload": f"fft1d_c2c_forward_n2^{t}", "n": 1 << t, "p": world,
         "input": "i.i.d. uniform [-1,1) re/im, SplitMix64 seed 0x08112535+t",
         "parallelism": ((f"reshape-transpose p={world} (" + ("fused NVLink push + 8 B NCCL barrier"
                                                              if exchange == "p2p" else "NCCL all-to-all")
                          + ")") if world > 1 else "single GPU"),
         "l2": (f"rank input of 16 n/p = {16 * (1 << t) / world / 2**20:.1f} MiB is not clearly larger than the 126 MB "
                "L2: a 512 MiB L2 flush (outside the timed events) before every timed step, step times summed")
               if l2_flush else
               (f"working set (in + out + scratch = {3 * 16 * (1 << t) // world >> 20} MiB per rank) larger than "
                "the 126 MB L2; no flush, K steps back to back in one event pair")}
    return c


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args, rank: int, world: int):
    import ctypes

    import torch
    import torch.distributed as dist

    import moa_inputs
    import paper_0811_2535_b200 as moa

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    t = args.t
    n = 1 << t
    if world > 1:
        moa.dist_init()
    M = n // world
    x = torch.empty(M, dtype=torch.complex128, device=dev)
    moa.gen_uniform(moa_inputs.seed_for(t), M, x, first=rank, stride=world)
    out = torch.empty_like(x)
    stream = torch.cuda.Stream(device=dev)
    plan = None
    if world > 1 and args.exchange in ("p2p", "auto"):
        # the fused NVLink exchange, admitted only if every rank reproduces the NCCL
        # path's result bit for bit (same arithmetic, only the transport differs)
        # every step that contains a collective runs only once all ranks agree the previous
        # one succeeded, so a failure on one rank cannot leave the others blocked in NCCL
        def agree(ok_local: int) -> bool:
            f = torch.tensor([ok_local], dtype=torch.int32, device=dev)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            return int(f.item()) == 1

        cand = None
        ok = 1
        try:
            cand = moa.Plan(n, world, -1, stream=stream, exchange=moa.XCHG_P2P)   # collective-free
        except Exception as e:  # noqa: BLE001 - any failure falls back to NCCL
            print(f"p2p plan unavailable ({e}); using NCCL", file=sys.stderr)
            ok = 0
        if agree(ok):
            try:
                cand.enable_p2p()                      # collective: handle all-gather
            except Exception as e:  # noqa: BLE001
                print(f"p2p mapping failed ({e}); using NCCL", file=sys.stderr)
                ok = 0
        else:
            ok = 0
        if agree(ok):
            try:
                ref_plan = moa.Plan(n, world, -1, stream=stream)
                with torch.cuda.stream(stream):
                    a = cand.execute(x)
                    b = ref_plan.execute(x)
                stream.synchronize()
                ok = int(torch.equal(a, b))
                ref_plan.destroy()
                del a, b
            except Exception as e:  # noqa: BLE001
                print(f"p2p exchange check failed ({e}); using NCCL", file=sys.stderr)
                ok = 0
        else:
            ok = 0
        if agree(ok):
            plan = cand
        else:
            if args.exchange == "p2p":
                raise RuntimeError("--exchange p2p: the fused exchange failed its bitwise check")
            if cand is not None:
                cand.destroy()
    exchange_used = "p2p" if plan is not None else "nccl"
    t_plan0 = time.perf_counter()
    if plan is None:
        plan = moa.Plan(n, world, -1, stream=stream)
    plan_ms = (time.perf_counter() - t_plan0) * 1e3   # plan creation: outside the timed region
    args.exchange = exchange_used
    info = plan.info()
    lib = moa.load()

    def barrier():
        if world > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            plan.execute(x, out)
    torch.cuda.synchronize()

    # ---- timed region: K steps, bracketed by CUDA events on the plan stream.  No event
    # sits between the kernels here: an event between two launches would serialise the
    # programmatic dependent launch the passes use (the next pass's CTAs are scheduled
    # while the previous pass drains).
    # When this rank's input is not clearly larger than the 126 MB L2 (p > 1: 2^24 / p), the
    # L2 is flushed (a 512 MiB write, outside the event pair) before every timed step and
    # the step times are summed; otherwise the K steps run back to back in one event pair.
    flush = 16 * M < 2 * L2_BYTES
    sampler = ClockSampler(dev.index)
    barrier()
    torch.cuda.synchronize()
    if flush:
        fl = torch.empty(1 << 27, dtype=torch.float32, device=dev)
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
        with sampler:
            with torch.cuda.stream(stream):
                for a, b in pairs:
                    fl.fill_(1.0)
                    a.record(stream)
                    plan.execute(x, out)
                    b.record(stream)
            pairs[-1][1].synchronize()
        torch.cuda.synchronize()
        barrier()
        elapsed = sum(a.elapsed_time(b) for a, b in pairs) * 1e-3
        del fl
    else:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with sampler:
            ev0.record(stream)
            for _ in range(args.steps):
                plan.execute(x, out)
            ev1.record(stream)
            ev1.synchronize()
        torch.cuda.synchronize()
        barrier()
        elapsed = ev0.elapsed_time(ev1) * 1e-3
    args.l2_flush = flush

    # ---- per-step spread (median / min / max) from K more steps with an event between steps
    step_evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    torch.cuda.synchronize()
    step_evs[0].record(stream)
    for i in range(args.steps):
        plan.execute(x, out)
        step_evs[i + 1].record(stream)
    step_evs[-1].synchronize()
    step_ms = sorted(step_evs[i].elapsed_time(step_evs[i + 1]) for i in range(args.steps))
    step_stats = {"median": round(statistics.median(step_ms), 4), "min": round(step_ms[0], 4),
                  "mean": round(statistics.mean(step_ms), 4), "max": round(step_ms[-1], 4)}

    # ---- the same K steps again with an event pair around every kernel (moa_fft_set_profiling):
    # per-kernel durations for the roofline line
    lib.moa_fft_set_profiling(plan._h, 1)
    stats_buf = (moa_stat * 16)()
    lib.moa_fft_get_profile(plan._h, stats_buf, 16)  # reset
    barrier()
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            plan.execute(x, out)
    nstat = lib.moa_fft_get_profile(plan._h, stats_buf, 16)
    lib.moa_fft_set_profiling(plan._h, 0)
    torch.cuda.synchronize()
    barrier()
    if world > 1:
        tt = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    value = args.steps * flops(n) / elapsed / 1e9
    kstats = [{"name": stats_buf[i].name.decode(), "launches": stats_buf[i].launches,
               "avg_us": stats_buf[i].total_ms * 1e3 / max(1, stats_buf[i].launches),
               "alg_bytes": int(stats_buf[i].alg_bytes)} for i in range(nstat)]
    kernel_total = sum(k["avg_us"] * k["launches"] for k in kstats if "NCCL" not in k["name"])
    kern = [k for k in kstats if "NCCL" not in k["name"]]
    dom = max(kern, key=lambda k: k["avg_us"] * k["launches"])
    peaks = measured_peaks()
    achieved = dom["alg_bytes"] / (dom["avg_us"] * 1e-6) / 1e9
    traffic = ncu_traffic(dom["name"], n, world)
    roofline = {"bound": "hbm", "kernel": dom["name"], "achieved": round(achieved, 1),
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                "traffic": traffic,
                "traffic_source": ("committed ncu --set full capture of this kernel (profiles/ncu_traffic.json), "
                                   "not measured in this run") if traffic is not None else None,
                "peak_source": peaks["source"],
                "share_of_step": round(dom["avg_us"] * dom["launches"] / max(kernel_total, 1e-9), 3),
                "kernel_timing": "per-kernel CUDA events on the plan stream over a second run of the same K "
                                 "steps (events between launches; the headline timed region has none)"}

    # ---- end to end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e and M > (1 << 27):
        # four pinned host buffers + four device staging buffers of n/p elements would
        # not fit host/device memory beside the timed buffers
        print(f"e2e skipped: n/p = 2^{M.bit_length() - 1} is beyond the pinned staging budget", file=sys.stderr)
    elif not args.no_e2e:
        # two pinned input/output pairs alternate: every step copies its whole input in
        # and its whole result out; the batch call overlaps those copies with the
        # transforms of the neighbouring steps (moa_fft_execute_host_batch)
        hins = [torch.from_numpy(moa_inputs.complex_signal(moa_inputs.seed_for(t), M, first=rank,
                                                           stride=world)).pin_memory() for _ in range(2)]
        houts = [torch.empty_like(hins[0]).pin_memory() for _ in range(2)]
        hin, hout = hins[0], houts[0]
        e_steps = max(2, min(args.steps, 20))
        plan.execute_host_batch(hins, houts)     # warm-up (allocates the staging pairs)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        plan.execute_host_batch([hins[i & 1] for i in range(e_steps)], [houts[i & 1] for i in range(e_steps)])
        t1.record(stream)
        t1.synchronize()
        e_el = t0.elapsed_time(t1) * 1e-3
        if world > 1:
            tt = torch.tensor([e_el], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_el = float(tt.item())
        e2e = {"value": round(e_steps * flops(n) / e_el / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": int(hin.numel() * 16), "d2h_bytes_per_step": int(hout.numel() * 16),
               "steps": e_steps, "ms_per_step": round(e_el / e_steps * 1e3, 3)}

    # ---- p > 1: no-overlap diagnostic of the exchange: the unchunked NCCL
    # plan (all-to-all on the plan stream, between the phase-1 passes and the combine)
    # with an event pair around every launch
    a2a = None
    if world > 1:
        try:
            a2a = a2a_diagnostic(moa, n, world, stream, x, args.steps, kstats, elapsed / args.steps, dev)
        except Exception as e:  # noqa: BLE001 - diagnostics never kill the bench line
            a2a = {"error": str(e)[:200]}

    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1:   # the oracle baseline: rank 0 at N = 1 only
            rate, cores, dt = cpu_oracle_rate(t, args.cpu_reps)
            cpu = {"value": round(rate, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{args.cpu_reps} full n=2^{t} oracle transforms ({dt:.2f} s each)",
                   "cpu": cpu_model()}
        step_s = elapsed / args.steps
        # SURVEY §8(d) algorithmic bytes: 32 n ceil(t/13) on one GPU (d(n) passes of <= 2^13
        # points); 32 M (d(M) + 1) per rank for p > 1 (the local passes + the P-point combine)
        M = n // world
        tm = M.bit_length() - 1
        survey_bytes = 32 * n * -(-t // 13) if world == 1 else 32 * M * (-(-tm // 13) + 1)
        hbm = {"alg_bytes_survey": int(survey_bytes),
               "alg_GBps_survey": round(survey_bytes / step_s / 1e9, 1),
               "frac_survey": round(survey_bytes / step_s / 1e9 / peaks["hbm_gbs"], 4),
               "survey_rule": "32 n ceil(t/13) (p = 1) / 32 (n/p)(d(n/p) + 1) per rank: the bytes of the "
                              "fewest <= 2^13-point passes (SURVEY §8(d)); the headline fraction",
               "alg_bytes_plan": int(info["hbm_bytes"]),
               "alg_GBps_plan": round(info["hbm_bytes"] / step_s / 1e9, 1),
               "frac_plan": round(info["hbm_bytes"] / step_s / 1e9 / peaks["hbm_gbs"], 4),
               "plan_rule": f"32 n x {info['passes']} passes of this plan's lifting {info['lift']} (its own "
                            "traffic; higher than the survey's when the plan makes more passes)",
               "peak_GBps": peaks["hbm_gbs"], "peak_source": peaks["source"]}
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
                "gpus_active": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(step_s * 1e3, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_block(t, world, info, args.exchange, getattr(args, "l2_flush", False)),
                "plan": {"lift": info["lift"], "passes": info["passes"], "chunks": info["chunks"],
                         "exchange": args.exchange if world > 1 else None},
                "hbm": hbm,
                "roofline": roofline, "kernels": kstats, "cpu_baseline": cpu, "e2e": e2e,
                "plan_ms": round(plan_ms, 2), "step_ms": step_stats,
                "gpu_launches": int(args.steps * info["launches"]),
                "clocks": sampler.summary()}
        if a2a is not None:
            line["a2a"] = a2a
        print(json.dumps(line), flush=True)
    plan.destroy()
    if world > 1:
        moa.dist_finalize()


def a2a_diagnostic(moa, n, world, stream, x, steps, kstats_main, step_s, dev):
    """Exchange cost without overlap (p > 1), max over ranks:
    t_a2a  = the NCCL send/recv group of the unchunked NCCL plan (events on the plan stream);
    algBw  = 16 M / t_a2a (this rank's buffer), busBw = algBw (p-1)/p (bytes that cross
             NVLink), as fractions of 900 GB/s nominal and 770 GB/s measured peer copy;
    fused  = for the P2P plan, the push pass minus the same pass storing locally (the
             NCCL plan's last pass): the exchange time the fused kernel adds;
    overlap efficiency = (t_p1 + t_a2a + t_p2 - t_step) / min(t_a2a, t_p1 + t_p2)."""
    import torch
    import torch.distributed as dist
    M = n // world
    ok = 1
    try:
        diag = moa.Plan(n, world, -1, stream=stream, chunks=1)
    except Exception:  # noqa: BLE001 - agree before any collective below
        ok = 0
    f = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(f, op=dist.ReduceOp.MIN)
    if int(f.item()) != 1:
        if ok:
            diag.destroy()
        return {"error": "diagnostic plan creation failed on some rank"}
    out = torch.empty_like(x)
    with torch.cuda.stream(stream):
        for _ in range(2):
            diag.execute(x, out)
    diag.set_profiling(True)
    diag.get_profile()
    dist.barrier()
    with torch.cuda.stream(stream):
        for _ in range(steps):
            diag.execute(x, out)
    prof = diag.get_profile()
    diag.set_profiling(False)
    torch.cuda.synchronize()
    diag.destroy()
    t_a2a = sum(k["avg_us"] for k in prof if "NCCL" in k["name"]) * 1e-6
    t_comb = sum(k["avg_us"] for k in prof if "pcombine" in k["name"]) * 1e-6
    t_p1 = sum(k["avg_us"] for k in prof if k["name"].startswith("pass")) * 1e-6
    last_local = max((k for k in prof if k["name"].startswith("pass")), key=lambda k: k["name"])["avg_us"] * 1e-6
    push = [k for k in kstats_main if "+push" in k["name"]]
    t_push_extra = (push[0]["avg_us"] * 1e-6 - last_local) if push else None
    vals = torch.tensor([t_a2a, t_p1, t_comb, t_push_extra if t_push_extra is not None else -1.0],
                        dtype=torch.float64, device=dev)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    t_a2a, t_p1, t_comb, t_push_extra = [float(v) for v in vals.tolist()]
    # reference: torch's own NCCL all_to_all_single on the same per-peer size (16 M / p bytes
    # per ordered pair), timed the same way -- the "measured NCCL all-to-all peak" of §8(d)
    sbuf = torch.empty(2 * M, dtype=torch.float64, device=dev)
    rbuf = torch.empty_like(sbuf)
    for _ in range(3):
        dist.all_to_all_single(rbuf, sbuf)
    torch.cuda.synchronize()
    dist.barrier()
    ra, rb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ra.record()
    for _ in range(steps):
        dist.all_to_all_single(rbuf, sbuf)
    rb.record()
    rb.synchronize()
    t_ref = torch.tensor([ra.elapsed_time(rb) * 1e-3 / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t_ref, op=dist.ReduceOp.MAX)
    t_ref = float(t_ref.item())
    del sbuf, rbuf
    alg = 16.0 * M / t_a2a / 1e9 if t_a2a > 0 else None
    bus = alg * (world - 1) / world if alg else None
    res = {"t_a2a_us": round(t_a2a * 1e6, 2), "t_phase1_us": round(t_p1 * 1e6, 2),
           "t_combine_us": round(t_comb * 1e6, 2), "bytes_sent_per_rank": int(16 * M // world * (world - 1)),
           "algBw_GBps": round(alg, 1) if alg else None, "busBw_GBps": round(bus, 1) if bus else None,
           "busBw_frac_of_900": round(bus / 900.0, 4) if bus else None,
           "busBw_frac_of_770_measured": round(bus / 770.0, 4) if bus else None,
           "nccl_a2a_ref_us": round(t_ref * 1e6, 2),
           "frac_of_nccl_a2a_ref": round(t_ref / t_a2a, 4) if t_a2a > 0 else None,
           "overlap_efficiency": round((t_p1 + t_a2a + t_comb - step_s) / min(t_a2a, t_p1 + t_comb), 4)
           if t_a2a > 0 else None,
           "how": "unchunked NCCL plan, events around every launch on the plan stream, max over ranks"}
    if t_push_extra is not None and t_push_extra > -1.0:
        res["fused_push_extra_us"] = round(t_push_extra * 1e6, 2)
        sent = 16.0 * M * (world - 1) / world
        if t_push_extra > 0:
            res["fused_push_GBps"] = round(sent / t_push_extra / 1e9, 1)
    return res


class moa_stat(__import__("ctypes").Structure):
    import ctypes as _c
    _fields_ = [("name", _c.c_char * 64), ("launches", _c.c_int), ("total_ms", _c.c_double),
                ("alg_bytes", _c.c_int64)]


def self_launch(n: int) -> int:
    """Re-run this command as n ranks: python -m torch.distributed.run --nproc-per-node n."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--t", type=int, default=24)
    ap.add_argument("--cpu-reps", type=int, default=5,
                    help="oracle transforms in the cpu_baseline sample (5 x 2^24 = about 11 s on 16 cores)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "p2p"],
                    help="p > 1 global transpose: NCCL send/recv group, or the last pass storing into the "
                         "peers' receive buffers over CUDA-IPC/NVLink (MOA_XCHG_P2P); auto = P2P when it "
                         "reproduces the NCCL result bitwise on every rank, else NCCL")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `bench.py --gpus N` without a launcher: start N ranks (one process per GPU) under
        # torch.distributed.run on this node and relay rank 0's line
        sys.exit(self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
