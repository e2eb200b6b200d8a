"""paper_0811_2535_b200 -- B200-native MoA reshape-transpose FFT (arXiv 0811.2535).

Thin ctypes binding over ``libmoa_fft.so`` (C ABI in ``include/moa_fft.h``).
It only marshals arguments: every step of the transform runs in the library's
CUDA kernels.  There is no CPU path: if the shared library is missing or
fails to load, importing this package raises.

    import torch, paper_0811_2535_b200 as moa
    X = moa.fft(x)                       # x: 1-D complex128 CUDA tensor, n = 2^t
    plan = moa.Plan(n, sign=-1)          # reusable plan
    plan.execute(x, out)
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

__all__ = ["Plan", "Plan2D", "PlanND", "fft2", "fftn", "fft", "dist_fft", "scatter_cyclic", "gather_cyclic", "ifft_unnormalized", "gen_uniform", "dist_init", "dist_finalize", "describe_pass",
           "Redist", "block_to_cyclic", "cyclic_to_block", "block_to_cyclic_via_central", "dist_fft_block",
           "LAYOUT_BLOCK", "LAYOUT_CYCLIC", "LAYOUT_CENTRAL", "ROUTE_DIRECT", "ROUTE_CENTRAL",
           "MoaError", "MODE_LIFTED", "MODE_LITERAL", "MODE_EMULATED", "XCHG_NCCL", "XCHG_P2P",
           "XCHG_P2P_EXTERNAL", "lib_path", "load"]

MODE_LIFTED, MODE_LITERAL, MODE_EMULATED = 0, 1, 2
XCHG_NCCL, XCHG_P2P, XCHG_P2P_EXTERNAL = 0, 1, 2
_ERRS = {-1: "INVALID_N", -2: "INVALID_P", -3: "INVALID_SIGN", -4: "ALIGN", -5: "NO_DIST",
         -6: "OOM", -7: "CUDA", -8: "NCCL", -9: "INVALID_ARG"}


class MoaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"MOA_ERR_{_ERRS.get(code, code)}: {msg}")
        self.code = code


class _Options(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("nlift", ctypes.c_int), ("lift", ctypes.c_int64 * 4),
                ("chunks", ctypes.c_int), ("exchange", ctypes.c_int), ("rank", ctypes.c_int),
                ("batch", ctypes.c_int64), ("breakpoint", ctypes.c_int)]


class _KernelStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 64), ("launches", ctypes.c_int), ("total_ms", ctypes.c_double),
                ("alg_bytes", ctypes.c_int64)]


class _Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("t", ctypes.c_int), ("p", ctypes.c_int), ("rank", ctypes.c_int),
                ("sign", ctypes.c_int), ("mode", ctypes.c_int), ("local_n", ctypes.c_int64),
                ("passes", ctypes.c_int), ("lift", ctypes.c_int64 * 4), ("breakpoint", ctypes.c_int),
                ("chunks", ctypes.c_int), ("launches", ctypes.c_int), ("workspace_bytes", ctypes.c_int64),
                ("hbm_bytes", ctypes.c_int64), ("a2a_bytes", ctypes.c_int64), ("batch", ctypes.c_int64)]


EXPORTS = ["moa_fft_plan", "moa_fft_plan_ex", "moa_fft_execute", "moa_fft_execute_host", "moa_fft_execute_host_batch",
           "moa_fft_destroy", "moa_fft_set_stream", "moa_fft_plan_info", "moa_fft_last_error",
           "moa_dist_unique_id", "moa_dist_init", "moa_dist_finalize", "moa_gen_uniform",
           "moa_fft_version", "moa_fft_set_profiling", "moa_fft_get_profile", "moa_fft_describe_pass",
           "moa_fft_ipc_handle", "moa_fft_ipc_open", "moa_fft_enable_p2p", "moa_fft_execute_phase",
           "moa_fft_plan_2d", "moa_fft_plan_nd", "moa_fft_default_lifting", "moa_fft_last_error_code",
           "moa_redist_plan", "moa_redist_execute", "moa_redist_set_stream", "moa_redist_info", "moa_redist_destroy"]

_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_needed: bool = True):
    """Load libmoa_fft.so, (re)building it with nvcc first when it is missing or older
    than any of its sources (build.needs_build), so a stale library is never loaded."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_needed and _build.needs_build():
        _build.build()
    if not os.path.exists(_build.LIB):
        raise ImportError(f"{_build.LIB} is missing; run paper_0811_2535_b200/build.py (no CPU fallback)")
    lib = ctypes.CDLL(_build.LIB, mode=ctypes.RTLD_GLOBAL)
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.moa_fft_plan.argtypes = [i64, ci, ci]
    lib.moa_fft_plan.restype = vp
    lib.moa_fft_plan_ex.argtypes = [i64, ci, ci, ctypes.POINTER(_Options)]
    lib.moa_fft_plan_ex.restype = vp
    lib.moa_fft_plan_2d.argtypes = [i64, i64, ci]
    lib.moa_fft_plan_2d.restype = vp
    lib.moa_fft_plan_nd.argtypes = [ci, vp, ci]
    lib.moa_fft_plan_nd.restype = vp
    lib.moa_fft_default_lifting.argtypes = [i64, ci, vp, ctypes.POINTER(ci)]
    lib.moa_fft_execute.argtypes = [vp, vp, vp]
    lib.moa_fft_execute_host.argtypes = [vp, vp, vp]
    lib.moa_fft_execute_host_batch.argtypes = [vp, ci, vp, vp]
    lib.moa_fft_ipc_handle.argtypes = [vp, vp]
    lib.moa_fft_ipc_open.argtypes = [vp, vp]
    lib.moa_fft_enable_p2p.argtypes = [vp]
    lib.moa_fft_execute_phase.argtypes = [vp, vp, vp, ci]
    lib.moa_fft_destroy.argtypes = [vp]
    lib.moa_fft_destroy.restype = None
    lib.moa_fft_set_stream.argtypes = [vp, vp]
    lib.moa_fft_plan_info.argtypes = [vp, ctypes.POINTER(_Info)]
    lib.moa_fft_last_error.restype = ctypes.c_char_p
    lib.moa_fft_last_error_code.restype = ctypes.c_int
    lib.moa_dist_unique_id.argtypes = [vp]
    lib.moa_dist_init.argtypes = [ci, ci, vp]
    lib.moa_gen_uniform.argtypes = [ctypes.c_uint64, i64, i64, i64, vp, vp]
    lib.moa_redist_plan.argtypes = [i64, ci, ci, ci, ci, ci]
    lib.moa_redist_plan.restype = vp
    lib.moa_redist_execute.argtypes = [vp, vp, vp]
    lib.moa_redist_set_stream.argtypes = [vp, vp]
    lib.moa_redist_info.argtypes = [vp, vp, vp, vp, vp]
    lib.moa_redist_destroy.argtypes = [vp]
    lib.moa_redist_destroy.restype = None
    lib.moa_fft_version.restype = ctypes.c_char_p
    lib.moa_fft_set_profiling.argtypes = [vp, ci]
    lib.moa_fft_get_profile.argtypes = [vp, vp, ci]
    lib.moa_fft_describe_pass.argtypes = [i64, ci, ci, ctypes.POINTER(_Options), ci, vp, vp, vp,
                                          ctypes.POINTER(i64)]
    _lib = lib
    return lib


def _err(code: int):
    raise MoaError(code, _lib.moa_fft_last_error().decode())


def _plan_err(lib):
    """A plan constructor returned NULL: raise with the library's own MOA_ERR_* code."""
    code = int(lib.moa_fft_last_error_code()) or -9
    raise MoaError(code, lib.moa_fft_last_error().decode())


def _ptr(x) -> int:
    return x if isinstance(x, int) else int(x.data_ptr())


def _cur_device():
    """The CUDA device plans bind to (torch's current device), None without CUDA."""
    try:
        import torch
        return int(torch.cuda.current_device()) if torch.cuda.is_available() else None
    except Exception:  # pragma: no cover
        return None


def _cur_stream() -> int:
    import torch
    return int(torch.cuda.current_stream().cuda_stream)


class Plan:
    """A reusable transform plan (moa_fft_plan_ex).

    n, p, sign: see include/moa_fft.h.  mode: MODE_LIFTED (product path),
    MODE_LITERAL (paper-literal bitrev + t radix-2 stages, ablation),
    MODE_EMULATED (p virtual ranks on one GPU).  lift: optional lifting <F1..Fd>.
    breakpoint (p > 1): 0 = the high end log2(n/p)+1, or log2(p)+1 = the low end
    (Fig 5.7's cyclic phase starts after the first log2 p stages; include/moa_fft.h).
    """

    def __init__(self, n: int, p: int = 1, sign: int = -1, mode: int = MODE_LIFTED,
                 lift=None, chunks: int = 0, stream=None, exchange: int = XCHG_NCCL, rank: int = 0,
                 batch: int = 1, breakpoint: int = 0):
        lib = load()
        opt = _Options()
        opt.mode = mode
        opt.breakpoint = breakpoint
        opt.chunks = chunks
        opt.exchange = exchange
        opt.rank = rank
        opt.batch = batch
        if lift:
            opt.nlift = len(lift)
            for i, f in enumerate(lift):
                opt.lift[i] = int(f)
        h = lib.moa_fft_plan_ex(int(n), int(p), int(sign), ctypes.byref(opt))
        if not h:
            _plan_err(lib)
        self._h = h
        self.device = _cur_device()
        self.n, self.p, self.sign, self.mode = int(n), int(p), int(sign), mode
        self.exchange, self.rank, self.batch = int(exchange), int(rank), max(1, int(batch))
        self._stream = None
        self.set_stream(stream)

    def set_stream(self, stream=None):
        """Bind to a stream (torch.cuda.Stream, raw handle int, or None = torch's current)."""
        if stream is None:
            s = _cur_stream()
        elif isinstance(stream, int):
            s = stream
        else:
            s = int(stream.cuda_stream)
        rc = _lib.moa_fft_set_stream(self._h, s)
        if rc:
            _err(rc)
        self._stream = s

    @property
    def stream(self) -> int:
        return self._stream

    def info(self) -> dict:
        inf = _Info()
        rc = _lib.moa_fft_plan_info(self._h, ctypes.byref(inf))
        if rc:
            _err(rc)
        d = {f: getattr(inf, f) for f, _ in _Info._fields_}
        d["lift"] = [int(v) for v in inf.lift[: inf.passes]] if self.mode != MODE_LITERAL else []
        return d

    def expected_elems(self) -> int:
        """Elements one execute reads and writes: batch*n (p = 1), n/p per rank, or all p
        ranks' slices back to back (EMULATED)."""
        if self.p == 1:
            return self.n * self.batch
        return self.n if self.mode == MODE_EMULATED else self.n // self.p

    def _check(self, x, what: str):
        """A tensor argument must be a contiguous complex128 CUDA tensor on the plan's
        device holding exactly expected_elems() elements (raw pointers are passed as is)."""
        if isinstance(x, int):
            return
        import torch
        if not isinstance(x, torch.Tensor):
            raise TypeError(f"{what} must be a torch tensor or a raw device pointer (int)")
        if x.dtype != torch.complex128:
            raise ValueError(f"{what} has dtype {x.dtype}; the transform is complex128")
        if not x.is_cuda or (self.device is not None and x.device.index != self.device):
            raise ValueError(f"{what} must live on cuda:{self.device} (got {x.device})")
        if not x.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        if x.numel() != self.expected_elems():
            raise ValueError(f"{what} holds {x.numel()} elements; this plan transforms {self.expected_elems()}")

    def execute(self, x, out=None):
        """Transform device data x (torch complex128 tensor or raw pointer) into out."""
        if out is None:
            import torch
            if isinstance(x, int):
                raise ValueError("out is required when x is a raw pointer")
            out = torch.empty_like(x)
        self._check(x, "x")
        self._check(out, "out")
        rc = _lib.moa_fft_execute(self._h, _ptr(x), _ptr(out))
        if rc:
            _err(rc)
        return out

    def execute_host(self, host_in, host_out):
        """End-to-end: host (ideally pinned) buffers in and out; synchronises."""
        rc = _lib.moa_fft_execute_host(self._h, _ptr(host_in), _ptr(host_out))
        if rc:
            _err(rc)
        return host_out

    def execute_host_batch(self, host_ins, host_outs):
        """Pipelined end-to-end: transform host_ins[i] into host_outs[i] (pinned host
        tensors), copies overlapping the transforms; synchronises."""
        k = len(host_ins)
        if len(host_outs) != k:
            raise ValueError("host_ins and host_outs differ in length")
        ins = (ctypes.c_void_p * max(k, 1))(*[_ptr(h) for h in host_ins])
        outs = (ctypes.c_void_p * max(k, 1))(*[_ptr(h) for h in host_outs])
        rc = _lib.moa_fft_execute_host_batch(self._h, k, ins, outs)
        if rc:
            _err(rc)
        return host_outs

    def ipc_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this rank's receive buffers (P2P plans)."""
        buf = (ctypes.c_char * 64)()
        rc = _lib.moa_fft_ipc_handle(self._h, buf)
        if rc:
            _err(rc)
        return bytes(buf)

    def ipc_open(self, handles):
        """Map every peer's receive buffers (handles: p 64-byte handles in rank order)."""
        blob = b"".join(handles)
        rc = _lib.moa_fft_ipc_open(self._h, ctypes.c_char_p(blob))
        if rc:
            _err(rc)

    def enable_p2p(self, group=None):
        """Exchange the IPC handles and map the peers.  With the library's NCCL
        communicator (MOA_XCHG_P2P) the library does it; otherwise (P2P_EXTERNAL)
        torch.distributed all-gathers the handles."""
        if self.exchange == XCHG_P2P:
            rc = _lib.moa_fft_enable_p2p(self._h)
            if rc:
                _err(rc)
            return
        import torch.distributed as dist
        hs = [None] * dist.get_world_size(group)
        dist.all_gather_object(hs, self.ipc_handle(), group=group)
        self.ipc_open(hs)

    def execute_phase(self, x, out, phase: int):
        """Phase 1 (local passes + fused push into the peers) or 2 (P-point combine)."""
        rc = _lib.moa_fft_execute_phase(self._h, _ptr(x) if x is not None else None,
                                        _ptr(out) if out is not None else None, int(phase))
        if rc:
            _err(rc)
        return out

    def set_profiling(self, enable: bool = True):
        """Bracket every kernel launch with CUDA events (moa_fft_set_profiling)."""
        rc = _lib.moa_fft_set_profiling(self._h, 1 if enable else 0)
        if rc:
            _err(rc)

    def get_profile(self) -> list:
        """Per-kernel event times since the last call (moa_fft_get_profile); resets them."""
        buf = (_KernelStat * 32)()
        k = _lib.moa_fft_get_profile(self._h, buf, 32)
        if k < 0:
            _err(k)
        return [{"name": buf[i].name.decode(), "launches": buf[i].launches,
                 "avg_us": buf[i].total_ms * 1e3 / max(1, buf[i].launches),
                 "alg_bytes": int(buf[i].alg_bytes)} for i in range(k)]

    def destroy(self):
        if getattr(self, "_h", None):
            _lib.moa_fft_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class Plan2D(Plan):
    """2-D transform of an n1 x n2 row-major complex128 array (moa_fft_plan_2d): the lifted
    1-D FFT over the rows, then one pass of n1-point DFTs over the columns (App. B's Omega)."""

    def __init__(self, n1: int, n2: int, sign: int = -1, stream=None):
        lib = load()
        h = lib.moa_fft_plan_2d(int(n1), int(n2), int(sign))
        if not h:
            _plan_err(lib)
        self._h = h
        self.device = _cur_device()
        self.n1, self.n2 = int(n1), int(n2)
        self.n, self.p, self.sign, self.mode = self.n1 * self.n2, 1, int(sign), MODE_LIFTED
        self.exchange, self.rank, self.batch = XCHG_NCCL, 0, 1
        self._stream = None
        self.set_stream(stream)


class PlanND(Plan):
    """r-D transform (r = 2, 3) of a row-major complex128 array (moa_fft_plan_nd): the lifted
    1-D FFT along the last axis, then one pass along each other axis (App. B's Omega)."""

    def __init__(self, shape, sign: int = -1, stream=None):
        lib = load()
        shp = (ctypes.c_int64 * len(shape))(*[int(v) for v in shape])
        h = lib.moa_fft_plan_nd(len(shape), shp, int(sign))
        if not h:
            _plan_err(lib)
        self._h = h
        self.device = _cur_device()
        self.shape = tuple(int(v) for v in shape)
        n = 1
        for v in self.shape:
            n *= v
        self.n, self.p, self.sign, self.mode = n, 1, int(sign), MODE_LIFTED
        self.exchange, self.rank, self.batch = XCHG_NCCL, 0, 1
        self._stream = None
        self.set_stream(stream)


def fftn(x, sign: int = -1, out=None):
    """2-D or 3-D transform of a complex128 CUDA tensor (row-major)."""
    import torch
    if x.dtype != torch.complex128 or not x.is_cuda or x.dim() not in (2, 3):
        raise ValueError("fftn expects a 2-D or 3-D complex128 CUDA tensor")
    x = x.contiguous()
    plan = PlanND(tuple(x.shape), sign)
    try:
        return plan.execute(x, out)
    finally:
        torch.cuda.current_stream().synchronize()
        plan.destroy()


def fft2(x, sign: int = -1, out=None):
    """2-D transform of a 2-D complex128 CUDA tensor (rows contiguous)."""
    import torch
    if x.dtype != torch.complex128 or not x.is_cuda or x.dim() != 2:
        raise ValueError("fft2 expects a 2-D complex128 CUDA tensor")
    x = x.contiguous()
    plan = Plan2D(x.shape[0], x.shape[1], sign)
    try:
        return plan.execute(x, out)
    finally:
        torch.cuda.current_stream().synchronize()
        plan.destroy()


def fft(x, sign: int = -1, out=None):
    """X_k = sum_j x_j exp(sign 2 pi i jk/n) of a 1-D complex128 CUDA tensor (n = 2^t)."""
    import torch
    if x.dtype != torch.complex128 or not x.is_cuda or x.dim() != 1:
        raise ValueError("fft expects a 1-D complex128 CUDA tensor")
    x = x.contiguous()
    plan = Plan(x.numel(), 1, sign)
    try:
        return plan.execute(x, out)
    finally:
        torch.cuda.current_stream().synchronize()
        plan.destroy()


def ifft_unnormalized(x, out=None):
    return fft(x, +1, out)


def gen_uniform(seed: int, count: int, out, first: int = 0, stride: int = 1, stream=None):
    """Fill a device buffer with the moa_inputs recipe (x_g = u(2g) + i u(2g+1), g = first + stride*i)."""
    lib = load()
    s = _cur_stream() if stream is None else (stream if isinstance(stream, int) else int(stream.cuda_stream))
    rc = lib.moa_gen_uniform(ctypes.c_uint64(seed), int(first), int(stride), int(count), _ptr(out), s)
    if rc:
        _err(rc)
    return out


def describe_pass(n: int, p: int, rank: int, pass_index: int, lift=None, breakpoint: int = 0):
    """Host-only index maps of one lifted pass (moa_fft_describe_pass; no GPU needed).

    Returns (F, in_idx, out_idx, tw_exp) as numpy int64 arrays of n/p entries."""
    import numpy as np
    lib = load()
    opt = _Options()
    opt.breakpoint = breakpoint
    if lift:
        opt.nlift = len(lift)
        for i, f in enumerate(lift):
            opt.lift[i] = int(f)
    m = n // p
    a, b, c = (np.empty(m, dtype=np.int64) for _ in range(3))
    F = ctypes.c_int64(0)
    rc = lib.moa_fft_describe_pass(int(n), int(p), int(rank), ctypes.byref(opt), int(pass_index),
                                   a.ctypes.data, b.ctypes.data, c.ctypes.data, ctypes.byref(F))
    if rc:
        _err(rc)
    return int(F.value), a, b, c


def dist_fft(x_local, n: int, sign: int = -1, out=None, exchange: int = XCHG_NCCL, breakpoint: int = 0):
    """One partitioned n-point transform over the torch.distributed world (after dist_init):
    x_local = x[rank::p] (complex128, this rank's GPU) -> X[rank::p] (the paper's xcyclic,
    P:799).  Collective: every rank calls it.  exchange = XCHG_P2P fuses the
    all-to-all into the last pass (the plan maps the peers' buffers first).  breakpoint:
    see Plan (both ends give the same X[rank::p])."""
    import torch
    import torch.distributed as dist
    p = dist.get_world_size()
    plan = Plan(n, p, sign, exchange=exchange, breakpoint=breakpoint)
    try:
        if exchange == XCHG_P2P:
            plan.enable_p2p()
        return plan.execute(x_local.contiguous(), out)
    finally:
        torch.cuda.current_stream().synchronize()
        plan.destroy()


LAYOUT_BLOCK, LAYOUT_CYCLIC, LAYOUT_CENTRAL = 0, 1, 2
ROUTE_DIRECT, ROUTE_CENTRAL = 0, 1


class Redist:
    """A redistribution between the paper's layouts of a distributed n-vector
    (moa_redist_plan, include/moa_fft.h): LAYOUT_BLOCK (rank r holds
    x[r*psize:(r+1)*psize]), LAYOUT_CYCLIC (x[r::p], the transform's layout) and
    LAYOUT_CENTRAL (all of x on rank 0).  route ROUTE_DIRECT = Fig 5.3/5.9 (one round,
    m(m-1) messages), ROUTE_CENTRAL = Fig 5.4 (gather to processor 0, scatter back).
    mode MODE_LIFTED = real ranks over the library's NCCL communicator (dist_init first),
    MODE_EMULATED = the p ranks' buffers back to back on this GPU."""

    def __init__(self, n: int, p: int, frm: int, to: int, route: int = ROUTE_DIRECT, mode: int = MODE_LIFTED,
                 stream=None):
        lib = load()
        h = lib.moa_redist_plan(int(n), int(p), int(frm), int(to), int(route), int(mode))
        if not h:
            _plan_err(lib)
        self._h = h
        self.n, self.p, self.frm, self.to, self.route, self.mode = int(n), int(p), int(frm), int(to), int(route), mode
        s = _cur_stream() if stream is None else (stream if isinstance(stream, int) else int(stream.cuda_stream))
        rc = lib.moa_redist_set_stream(h, s)
        if rc:
            _err(rc)

    def info(self) -> dict:
        m, b, ei, eo = (ctypes.c_int64() for _ in range(4))
        rc = _lib.moa_redist_info(self._h, ctypes.byref(m), ctypes.byref(b), ctypes.byref(ei), ctypes.byref(eo))
        if rc:
            _err(rc)
        return {"messages": m.value, "max_rank_bytes": b.value, "elems_in": ei.value, "elems_out": eo.value}

    def execute(self, x, out=None):
        """x: this rank's elements (complex128 CUDA tensor, or None where the layout gives
        the rank none); returns out (allocated when None)."""
        import torch
        inf = self.info()
        if out is None and inf["elems_out"] > 0:
            dev = x.device if x is not None else torch.device("cuda", torch.cuda.current_device())
            out = torch.empty(inf["elems_out"], dtype=torch.complex128, device=dev)
        for v, k, what in ((x, "elems_in", "x"), (out, "elems_out", "out")):
            if v is not None and (v.dtype != torch.complex128 or not v.is_cuda or not v.is_contiguous()
                                  or v.numel() != inf[k]):
                raise ValueError(f"{what} must be a contiguous complex128 CUDA tensor of {inf[k]} elements")
        rc = _lib.moa_redist_execute(self._h, _ptr(x) if x is not None else None,
                                     _ptr(out) if out is not None else None)
        if rc:
            _err(rc)
        return out

    def destroy(self):
        if getattr(self, "_h", None):
            _lib.moa_redist_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def _redist(x, n: int, frm: int, to: int, route: int = ROUTE_DIRECT):
    """One redistribution over the library's communicator (collective; dist_init first)."""
    import torch
    import torch.distributed as dist
    plan = Redist(n, dist.get_world_size(), frm, to, route)
    try:
        return plan.execute(x)
    finally:
        torch.cuda.current_stream().synchronize()
        plan.destroy()


def scatter_cyclic(x0, n: int):
    """The paper's DISTRIBUTE_CENTRALIZED_TO_CYCLIC_PARTITIONED (Fig 5.8):
    rank 0 holds x0 (n elements, CUDA), rank r receives x0[r::p].  Library pack kernel +
    NCCL scatter; other ranks pass None."""
    return _redist(x0, n, LAYOUT_CENTRAL, LAYOUT_CYCLIC)


def gather_cyclic(xcyclic, n: int):
    """DISTRIBUTE_CYCLIC_PARTITIONED_TO_CENTRALIZED (Fig 5.8): rank r holds
    X[r::p]; rank 0 returns the whole n-vector in natural order, the others None."""
    return _redist(xcyclic, n, LAYOUT_CYCLIC, LAYOUT_CENTRAL)


def block_to_cyclic(x_block, n: int = None, route: int = ROUTE_DIRECT):
    """Natural block x[r*psize:(r+1)*psize] -> x[r::p]: Fig 5.3/5.9's direct exchange
    (route ROUTE_DIRECT) or Fig 5.4 through processor 0 (ROUTE_CENTRAL)."""
    import torch.distributed as dist
    n = n or x_block.numel() * dist.get_world_size()
    return _redist(x_block, n, LAYOUT_BLOCK, LAYOUT_CYCLIC, route)


def cyclic_to_block(x_cyclic, n: int = None, route: int = ROUTE_DIRECT):
    """x[r::p] -> the natural block x[r*psize:(r+1)*psize] (the transform's output to
    block-natural order)."""
    import torch.distributed as dist
    n = n or x_cyclic.numel() * dist.get_world_size()
    return _redist(x_cyclic, n, LAYOUT_CYCLIC, LAYOUT_BLOCK, route)


def block_to_cyclic_via_central(x_block, n: int = None):
    """Fig 5.4: the block -> cyclic redistribution routed through
    processor 0 (2(m-1) messages, every element moved twice)."""
    return block_to_cyclic(x_block, n, ROUTE_CENTRAL)


def dist_fft_block(x_block, n: int, sign: int = -1, exchange: int = XCHG_NCCL, breakpoint: int = 0):
    """One partitioned transform with NATURAL block layouts in and out: rank r
    holds x[r*psize : (r+1)*psize] and returns X[r*psize : (r+1)*psize].  = block_to_cyclic
    -> dist_fft -> cyclic_to_block: the transform's own exchange plus two layout
    all-to-alls (torch.distributed; collective)."""
    xc = block_to_cyclic(x_block, n)
    return cyclic_to_block(dist_fft(xc, n, sign, exchange=exchange, breakpoint=breakpoint), n)


def default_lifting(n: int, p: int = 1) -> list:
    """The plan builder's default lifting <F1..Fd> of n/p (host only, no GPU)."""
    lib = load()
    lift = (ctypes.c_int64 * 4)()
    d = ctypes.c_int(0)
    rc = lib.moa_fft_default_lifting(int(n), int(p), lift, ctypes.byref(d))
    if rc:
        _err(rc)
    return [int(lift[i]) for i in range(d.value)]


def bcast_unique_id(group=None) -> bytes:
    """Rank 0 creates an ncclUniqueId (moa_dist_unique_id); torch.distributed broadcasts it."""
    import torch
    import torch.distributed as dist
    lib = load()
    rank = dist.get_rank(group)
    buf = (ctypes.c_char * 128)()
    if rank == 0:
        rc = lib.moa_dist_unique_id(buf)
        if rc:
            _err(rc)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    t = torch.frombuffer(bytearray(bytes(buf)), dtype=torch.uint8).to(dev)
    dist.broadcast(t, 0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def dist_init(group=None):
    """Create the library's NCCL communicator over torch.distributed's world."""
    import torch.distributed as dist
    lib = load()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ident = bcast_unique_id(group)
    rc = lib.moa_dist_init(rank, world, ctypes.c_char_p(ident))
    if rc:
        _err(rc)
    return rank, world


def dist_finalize():
    load().moa_dist_finalize()
