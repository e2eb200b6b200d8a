"""Host logic of the plan builder, checked on the CPU (no GPU needed).

moa_fft_describe_pass exposes, for every lifted pass, the exact index maps and
twiddle exponents the CUDA pass kernel uses (same PassDesc, same address
arithmetic).  Replaying those maps with numpy's FFT for the F-point inner
transforms must reproduce the oracle: this pins the lifting (reshape), the
transposed store (Fig A.1 transpose+ravel), the inter-pass twiddles
and, for p > 1, the rank twiddle + pack of Fig 4.4/5.9 and the cyclic output
layout X[r + p*i].  The arithmetic here is test-side numpy;
what is under test is the product's host-side index logic.
"""
import numpy as np
import pytest

import moa_inputs
import oracle
import paper_0811_2535_b200 as moa


def replay_local(x_local, n, p, rank, lift=None, breakpoint=0):
    """Run the local passes of one rank from their maps (numpy arithmetic)."""
    m = n // p
    k = 0
    cur = np.asarray(x_local, dtype=np.complex128)
    while True:
        try:
            F, ii, oi, tw = moa.describe_pass(n, p, rank, k, lift, breakpoint)
        except moa.MoaError as e:
            if "outside" in str(e) and k > 0:
                break
            raise
        assert np.array_equal(np.sort(ii), np.arange(m)), "input map is not a permutation"
        assert np.array_equal(np.sort(oi), np.arange(m)), "output map is not a permutation"
        y = np.fft.fft(cur[ii].reshape(-1, F), axis=1).reshape(-1)
        sel = tw >= 0
        y[sel] *= np.exp(-2j * np.pi * (tw[sel].astype(np.float64) / n))
        nxt = np.empty(m, dtype=np.complex128)
        nxt[oi] = y
        cur = nxt
        k += 1
    return cur


def pcombine(recv, p):
    """out[c + chunk*k2] = sum_s omega_p^(s*k2) recv[s*chunk + c] (Fig 5.7 cyclic phase, lifted)."""
    chunk = recv.size // p
    R = recv.reshape(p, chunk)
    return np.fft.fft(R, axis=0).reshape(-1)


@pytest.mark.parametrize("t,lift", [
    (4, None), (10, None), (13, None), (14, None), (16, None), (20, None), (22, None),
    (12, [64, 64]), (16, [16, 16, 256]), (18, [8, 32, 1024]), (20, [16, 16, 16, 256]),
    (20, [1024, 1024]), (24, [256, 256, 256]), (24, [4096, 4096]),
])
def test_single_rank_maps_compose_to_fft(t, lift):
    n = 1 << t
    x = moa_inputs.signal_for(t)
    got = replay_local(x, n, 1, 0, lift)
    assert oracle.rel_l2(got, oracle.fft(x, -1, threads=8)) <= 1e-13


@pytest.mark.parametrize("t,p,lift", [(6, 2, None), (8, 8, None), (10, 4, None), (14, 2, None),
                                      (16, 8, None), (20, 4, None), (21, 4, [32, 128, 128]),
                                      (18, 8, [8, 32, 128])])
def test_partitioned_maps_with_exchange(t, p, lift):
    """Every rank's phase 1 from its maps, the Fig 5.9 exchange, then the P-point combine."""
    n = 1 << t
    x = moa_inputs.signal_for(t)
    ref = oracle.fft(x, -1, threads=8)
    m = n // p
    chunk = m // p
    send = [replay_local(x[r::p], n, p, r, lift) for r in range(p)]
    for d in range(p):
        recv = np.concatenate([send[s][d * chunk:(d + 1) * chunk] for s in range(p)])
        out = pcombine(recv, p)
        assert oracle.rel_l2(out, ref[d::p]) <= 1e-13, (d, p)


def psplit(x_local, n, p, r):
    """Low-end phase 1 (test-side numpy): P-point DFTs over x_local[c + chunk*s], times
    omega_n^((r + p*c)*u), send layout [u][c]."""
    chunk = x_local.size // p
    Z = np.fft.fft(np.asarray(x_local).reshape(p, chunk), axis=0)
    e = ((r + p * np.arange(chunk))[None, :] * np.arange(p)[:, None]) % n
    return (Z * np.exp(-2j * np.pi * e / n)).reshape(-1)


@pytest.mark.parametrize("t,p", [(3, 2), (8, 2), (10, 4), (14, 2), (16, 8), (16, 16), (20, 4)])
def test_low_end_breakpoint_decomposition(t, p):
    """The arithmetic the low-end kernels implement (Fig 5.7, breakpoint = log2 p + 1,
    P:665), in numpy: psplit (P-point DFTs over x_local[c + chunk*s] + the
    weightcyclic factor omega_n^((r + p*c)*u)), the Fig 5.9 exchange, the p FFTs of
    length n/p^2 of the received [source][c] blocks, the factor omega_{n/p}^(s*c) and
    the p-point DFT over s -- X[u + p*v] on rank u, the same as the high end."""
    n = 1 << t
    x = moa_inputs.signal_for(t)
    ref = oracle.fft(x, -1, threads=8)
    m = n // p
    chunk = m // p
    send = [psplit(x[r::p], n, p, r) for r in range(p)]
    for u in range(p):
        recv = np.stack([send[s][u * chunk:(u + 1) * chunk] for s in range(p)])   # [s][c]
        blocks = np.fft.fft(recv, axis=1)
        blocks *= np.exp(-2j * np.pi * (np.arange(p)[:, None] * np.arange(chunk)[None, :] % m) / m)
        got = np.fft.fft(blocks, axis=0).reshape(-1)                               # out[c + chunk*k]
        assert oracle.rel_l2(got, ref[u::p]) <= 1e-13, (u, p)


def test_breakpoint_validation():
    n = 1 << 12
    with pytest.raises(moa.MoaError, match="breakpoint"):
        moa.describe_pass(n, 4, 0, 0, None, 5)        # interior breakpoints are oracle-only
    with pytest.raises(moa.MoaError, match="breakpoint"):
        moa.describe_pass(n, 1, 0, 0, None, 1)        # p = 1 has no cyclic phase
    moa.describe_pass(n, 4, 0, 0, None, 11)           # log2(psize) + 1 = the default
    with pytest.raises(moa.MoaError, match="batched"):
        moa.describe_pass(n, 4, 0, 0, None, 3)        # the low end runs a batched p = 1 plan
    moa.describe_pass(16, 4, 0, 0, None, 3)           # psize = p: both ends are log2 p + 1


def test_column_pass_reads_contiguous_runs():
    # middle/first passes read T adjacent columns: runs of T contiguous elements
    F, ii, _, _ = moa.describe_pass(1 << 24, 1, 0, 0)
    rows = ii.reshape(-1, F)            # one row per transform
    T = 16
    assert np.all(np.diff(rows[:T, 0]) == 1)   # T transforms of a tile = T adjacent columns


def test_describe_pass_validation():
    with pytest.raises(moa.MoaError):
        moa.describe_pass(100, 1, 0, 0)
    with pytest.raises(moa.MoaError):
        moa.describe_pass(1 << 10, 1, 0, 5)
    with pytest.raises(moa.MoaError):
        moa.describe_pass(1 << 10, 4, 4, 0)


def test_default_lifting_table_every_t_and_p():
    """SURVEY §4.2 'lifting table for every t and P': the default lifting of n/p is a
    factorisation into powers of two in [2, 2^13], at most 4 levels (3 when p > 1, the
    pack layout's tile dimensions), first factor >= p for multi-level p > 1 plans, and
    the documented table entries."""
    for t in range(1, 33):
        for p in (1, 2, 4, 8):
            n = 1 << t
            if n // p < p:
                with pytest.raises(moa.MoaError):
                    moa.default_lifting(n, p)
                continue
            lift = moa.default_lifting(n, p)
            prod = 1
            for f in lift:
                assert f >= 2 and f <= 8192 and f & (f - 1) == 0, (t, p, lift)
                prod *= f
            assert prod == n // p, (t, p, lift)
            assert len(lift) <= (3 if p > 1 else 4), (t, p, lift)
            if p > 1 and len(lift) > 1:
                assert lift[0] >= p, (t, p, lift)
    assert moa.default_lifting(1 << 24) == [256, 256, 256]
    assert moa.default_lifting(1 << 20) == [256, 4096]
    assert moa.default_lifting(1 << 15) == [256, 128]
    assert moa.default_lifting(1 << 21, 2) == [1024, 1024]   # p > 1 keeps <2^(tl/2), 2^(tl/2)>
    assert moa.default_lifting(1 << 21) == [128, 256, 64]
    assert moa.default_lifting(1 << 22) == [128, 256, 128]
    assert moa.default_lifting(1 << 23) == [128, 256, 256]
    assert moa.default_lifting(1 << 26) == [256, 256, 1024]
    assert moa.default_lifting(1 << 30) == [128, 128, 256, 256]
    assert moa.default_lifting(1 << 29) == [128, 128, 128, 256]
    assert moa.default_lifting(1 << 10) == [1024]
    assert moa.default_lifting(1 << 30, 2) == [256, 512, 4096]   # per rank 2^29 (profiles/r02_lifting_recheck.md)
    assert moa.default_lifting(1 << 30, 8) == [256, 256, 2048]   # configs[3]'s per-rank plan
    assert moa.default_lifting(1 << 31, 2) == [512, 512, 4096]
