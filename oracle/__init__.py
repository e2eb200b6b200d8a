"""CPU oracle for the MoA reshape-transpose FFT -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product path
(``paper_0811_2535_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``oracle/moa_oracle.c`` (plain C, built with
``-O2 -ffp-contract=off -fno-fast-math -fopenmp``).  Each function names the
paper figure it follows (P:<line> of PAPER.md, arXiv 0811.2535):

* ``fft``       -- Fig 2.1 in the Fig 3.9 in-place form;
                   ``threads > 1`` is the Fig 6.1 ``parallel do`` template
* ``fft_temp``  -- Fig 3.8, temporary ``xx``
* ``dft``       -- the plain definition X_k = sum_j x_j w^{jk}, O(n^2), long double
* ``dft_bins``  -- the same definition at selected bins (sampled parity at large n)
* ``dft_bins_range`` -- its sum over one window x[j0 : j0+len] (windows of a partition add
                   up to ``dft_bins``; streams inputs larger than host memory)
* ``bitrev``    -- P_n, Fig 2.1 line 1
* ``weights``   -- weight(row) = EXP(sign 2 pi i row / L) (Fig 3.8)
* ``dist_sim``  -- Fig 5.7 + Fig 5.9 with m virtual processors
* ``gamma``     -- row-major offset, Def A.1
* ``fft2``      -- 2-D DFT as App. B's Omega: (fft Omega <1>) over the rows, transpose
                   (Fig A.1), (fft Omega <1>) again, transpose back (B.1-B.6)
* ``dft2``      -- the plain 2-D definition, O((n1 n2)^2), for pinning ``fft2``
* ``fftn``      -- r-D DFT via Omega: ``fft`` along every axis in turn (last axis first)
* ``dftn``      -- the plain r-D definition (tiny arrays), for pinning ``fftn``
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "moa_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (gcc); returns its path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            dp = ctypes.POINTER(ctypes.c_double)
            i64 = ctypes.c_int64
            lib.oracle_fft.argtypes = [i64, ctypes.c_int, ctypes.c_int, dp, dp]
            lib.oracle_fft_temp.argtypes = [i64, ctypes.c_int, dp, dp]
            lib.oracle_dft.argtypes = [i64, ctypes.c_int, dp, dp]
            lib.oracle_dft_bins.argtypes = [i64, ctypes.c_int, dp, i64, ctypes.POINTER(i64), dp]
            lib.oracle_dft_bins_range.argtypes = [i64, ctypes.c_int, dp, i64, i64, i64, ctypes.POINTER(i64), dp]
            lib.oracle_bitrev.argtypes = [i64, dp, dp]
            lib.oracle_weights.argtypes = [i64, ctypes.c_int, dp]
            lib.oracle_omega.argtypes = [i64, i64, ctypes.c_int, dp]
            lib.oracle_omega.restype = None
            lib.oracle_rev.argtypes = [i64, ctypes.c_int]
            lib.oracle_rev.restype = i64
            lib.oracle_dist_sim.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp,
                                            dp, ctypes.POINTER(i64)]
            lib.oracle_gamma.argtypes = [ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]
            lib.oracle_gamma.restype = i64
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def fft(x, sign: int = -1, threads: int = 1) -> np.ndarray:
    x = _c128(x)
    out = np.empty_like(x)
    _check(_load().oracle_fft(x.size, sign, threads, _dp(x), _dp(out)), "fft")
    return out


def fft_temp(x, sign: int = -1) -> np.ndarray:
    x = _c128(x)
    out = np.empty_like(x)
    _check(_load().oracle_fft_temp(x.size, sign, _dp(x), _dp(out)), "fft_temp")
    return out


def dft(x, sign: int = -1) -> np.ndarray:
    x = _c128(x)
    out = np.empty_like(x)
    _check(_load().oracle_dft(x.size, sign, _dp(x), _dp(out)), "dft")
    return out


def dft_bins(x, ks, sign: int = -1) -> np.ndarray:
    """X_k of the plain definition at the listed bins only (any power-of-two n)."""
    x = _c128(x)
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.int64))
    out = np.empty(ks.size, dtype=np.complex128)
    lib = _load()
    rc = lib.oracle_dft_bins(x.size, sign, _dp(x), ks.size,
                             ks.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(out))
    _check(rc, "dft_bins")
    return out


def dft_bins_range(x_window, n: int, j0: int, ks, sign: int = -1) -> np.ndarray:
    """The plain definition restricted to x[j0 : j0 + len(x_window)]: summing the
    windows of a partition of [0, n) gives dft_bins (inputs too large for host memory)."""
    x = _c128(x_window)
    ks = np.ascontiguousarray(np.asarray(ks, dtype=np.int64))
    out = np.empty(ks.size, dtype=np.complex128)
    rc = _load().oracle_dft_bins_range(int(n), sign, _dp(x), int(j0), x.size, ks.size,
                                       ks.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(out))
    _check(rc, "dft_bins_range")
    return out


def bitrev(x) -> np.ndarray:
    x = _c128(x)
    out = np.empty_like(x)
    _check(_load().oracle_bitrev(x.size, _dp(x), _dp(out)), "bitrev")
    return out


def rev(j: int, t: int) -> int:
    return int(_load().oracle_rev(j, t))


def weights(L: int, sign: int = -1) -> np.ndarray:
    out = np.empty(max(L // 2, 1), dtype=np.complex128)
    _check(_load().oracle_weights(L, sign, _dp(out)), "weights")
    return out[: L // 2]


def omega(e: int, L: int, sign: int = -1) -> complex:
    out = np.empty(1, dtype=np.complex128)
    _load().oracle_omega(e, L, sign, _dp(out))
    return complex(out[0])


def dist_sim(x, m: int, breakpoint: int | None = None, sign: int = -1):
    """Fig 5.7/5.9 simulation.  Returns (xcyclic[m, psize], gathered X[n], counts dict).

    breakpoint defaults to the high end log2(psize)+1 (reading R6)."""
    x = _c128(x)
    n = x.size
    psize = n // m
    if breakpoint is None:
        breakpoint = int(psize).bit_length()  # log2(psize) + 1
    cyc = np.empty(n, dtype=np.complex128)
    out = np.empty(n, dtype=np.complex128)
    counts = (ctypes.c_int64 * 4)()
    _check(_load().oracle_dist_sim(n, m, breakpoint, sign, _dp(x), _dp(cyc), _dp(out), counts),
           "dist_sim")
    c = {"messages": counts[0], "elements_per_message": counts[1],
         "weights_per_proc": counts[2], "assigns_per_stage": counts[3]}
    return cyc.reshape(m, psize), out, c


def gamma(shape, index) -> int:
    d = len(shape)
    s = (ctypes.c_int64 * d)(*shape)
    i = (ctypes.c_int64 * d)(*index)
    return int(_load().oracle_gamma(d, s, i))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def l2_parts(got, ref, chunk: int = 1 << 22):
    """(sum |g-o|^2, sum |o|^2) accumulated in long double, chunked so 2^30 fits in RAM."""
    g = np.ascontiguousarray(got, dtype=np.complex128).reshape(-1).view(np.float64)
    o = np.ascontiguousarray(ref, dtype=np.complex128).reshape(-1).view(np.float64)
    if g.shape != o.shape:
        raise ValueError(f"shape mismatch {g.shape} vs {o.shape}")
    num = np.longdouble(0)
    den = np.longdouble(0)
    for s in range(0, g.size, chunk):
        gg = g[s:s + chunk].astype(np.longdouble)
        oo = o[s:s + chunk].astype(np.longdouble)
        num += np.sum((gg - oo) ** 2)
        den += np.sum(oo ** 2)
    return num, den


def rel_l2(got, ref) -> float:
    """relL2 = ||g - o||_2 / ||o||_2 accumulated in long double."""
    num, den = l2_parts(got, ref)
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))


def fft2(x, sign: int = -1, threads: int = 1) -> np.ndarray:
    """2-D DFT of an n1 x n2 array via App. B's Omega.

    (f Omega <1>) xi applies f to every 1-D sub-array i psi xi along the last axis
    (B.4-B.6): step 1 the rows, step 2 the transpose of Fig A.1, step 3 the rows of
    the transpose (= the columns), step 4 the transpose back.  f = ``fft`` (Fig 3.9)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    if a.ndim != 2:
        raise ValueError("fft2 expects a 2-D array")
    y = np.stack([fft(row, sign, threads) for row in a])            # (fft Omega <1>) x
    z = np.ascontiguousarray(y.T)                                    # transpose
    w = np.stack([fft(row, sign, threads) for row in z])            # (fft Omega <1>) z
    return np.ascontiguousarray(w.T)                                 # transpose back


def dft2(x, sign: int = -1) -> np.ndarray:
    """X[k1,k2] = sum_{j1,j2} x[j1,j2] exp(sign 2 pi i (j1 k1/n1 + j2 k2/n2)), written out
    as the double sum in long double with exactly reduced exponents (tiny arrays only)."""
    a = np.asarray(x, dtype=np.complex128)
    n1, n2 = a.shape
    out = np.empty((n1, n2), dtype=np.complex128)
    ld = np.longdouble
    for k1 in range(n1):
        for k2 in range(n2):
            re = ld(0)
            im = ld(0)
            for j1 in range(n1):
                for j2 in range(n2):
                    # angle as an exact fraction of a turn: (j1 k1 n2 + j2 k2 n1) / (n1 n2)
                    e = (j1 * k1 * n2 + j2 * k2 * n1) % (n1 * n2)
                    th = ld(sign) * ld(2) * ld(np.pi) * ld(e) / ld(n1 * n2)
                    c, s_ = np.cos(th), np.sin(th)
                    xr, xi = ld(a[j1, j2].real), ld(a[j1, j2].imag)
                    re += xr * c - xi * s_
                    im += xr * s_ + xi * c
            out[k1, k2] = complex(float(re), float(im))
    return out


def fftn(x, sign: int = -1, threads: int = 1) -> np.ndarray:
    """r-D DFT via App. B's Omega: for each axis a (last first), move axis a last
    (a transpose, Fig A.1), apply (fft Omega <1>) to every 1-D sub-array (B.4-B.6),
    move it back.  f = ``fft`` (Fig 3.9)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    for ax in range(a.ndim - 1, -1, -1):
        m = np.ascontiguousarray(np.moveaxis(a, ax, -1))
        flat = m.reshape(-1, m.shape[-1])
        res = np.stack([fft(row, sign, threads) for row in flat]).reshape(m.shape)
        a = np.ascontiguousarray(np.moveaxis(res, -1, ax))
    return a


def dftn(x, sign: int = -1) -> np.ndarray:
    """The r-D definition written out as one sum over all index tuples (long double,
    exponents reduced exactly modulo the array size); tiny arrays only."""
    a = np.asarray(x, dtype=np.complex128)
    shape = a.shape
    N = int(np.prod(shape))
    idx = list(np.ndindex(*shape))
    out = np.empty(shape, dtype=np.complex128)
    ld = np.longdouble
    for k in idx:
        re = ld(0)
        im = ld(0)
        for j in idx:
            e = sum(j[d] * k[d] * (N // shape[d]) for d in range(len(shape))) % N
            th = ld(sign) * ld(2) * ld(np.pi) * ld(e) / ld(N)
            c, s_ = np.cos(th), np.sin(th)
            xr, xi = ld(a[j].real), ld(a[j].imag)
            re += xr * c - xi * s_
            im += xr * s_ + xi * c
        out[k] = complex(float(re), float(im))
    return out
