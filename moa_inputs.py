"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no FFT, twiddle or index map):
only the counter-based generator that both sides use to build identical
inputs (SURVEY.md §8(d) "Inputs").

SplitMix64 of (seed, global index):
    z = seed + (idx + 1) * 0x9E3779B97F4A7C15
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB
    z ^= z >> 31
    u = (z >> 11) * 2^-52 - 1           # exact in double, uniform on [-1, 1)
Complex element g of the length-n signal: x_g = u(seed, 2g) + i*u(seed, 2g + 1).
seed_t = 0x08112535 + t for n = 2^t; the second vector of a linearity check
uses seed_t + 0x1000.  Because the generator is index-addressed, rank r of P
can generate its residue class x[r + P*j] alone, and the CUDA twin
(moa_gen_uniform in the product library) reproduces these values bit for bit.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 0x08112535
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def seed_for(t: int, second: bool = False) -> int:
    return SEED_BASE + t + (0x1000 if second else 0)


def splitmix64(seed: int, idx) -> np.ndarray:
    """Raw 64-bit SplitMix64 output for (seed, idx)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, idx) -> np.ndarray:
    """u(seed, idx) in [-1, 1) for an array of uint64 indices."""
    z = splitmix64(seed, idx)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def complex_signal(seed: int, count: int, first: int = 0, stride: int = 1,
                   chunk: int = 1 << 22) -> np.ndarray:
    """x_g for g = first + stride*i, i < count, as complex128 (chunked)."""
    out = np.empty(count, dtype=np.complex128)
    f = out.view(np.float64)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        g = np.uint64(first) + np.uint64(stride) * np.arange(s, e, dtype=np.uint64)
        f[2 * s:2 * e:2] = uniform(seed, np.uint64(2) * g)
        f[2 * s + 1:2 * e:2] = uniform(seed, np.uint64(2) * g + np.uint64(1))
    return out


def signal_for(t: int, second: bool = False) -> np.ndarray:
    """The full length-2^t benchmark/parity input."""
    return complex_signal(seed_for(t, second), 1 << t)


def rank_slice(t: int, rank: int, p: int, second: bool = False) -> np.ndarray:
    """Rank r's cyclic input a_r[j] = x[r + p*j]."""
    n = 1 << t
    return complex_signal(seed_for(t, second), n // p, first=rank, stride=p)
