"""Pins for the CPU oracle (SURVEY.md §8(c) "What pins each part").

Every check ties the oracle to something other than itself: worked values
(tests/golden/, each cited), closed forms, invariants of the DFT, special
cases reducing to library routines (numpy.fft / pocketfft, the clongdouble
FFT), brute force on tiny inputs, and the paper's structural counts.  A
plausible mistake anywhere in the oracle (a dropped term, wrong sign, wrong
index, transposed operand, wrong weight) fails at least one of them.
"""
import math
import os

import numpy as np
import pytest

import moa_inputs
import oracle
from conftest import parse_complex_list, read_golden

SIGNS = (-1, 1)


def _rand(n, seed=1234):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


# ---------------------------------------------------------------- worked values
def test_worked_values(golden_dir):
    rows = read_golden(os.path.join(golden_dir, "worked_values.txt"))
    assert len(rows) >= 9
    for kind, sign, inp, exp in rows:
        if kind == "fft":
            x = parse_complex_list(inp)
            want = np.array(parse_complex_list(exp))
            for f in (oracle.fft, oracle.fft_temp, oracle.dft):
                got = f(x, int(sign))
                assert np.max(np.abs(got - want)) <= 1e-15, (f.__name__, x, got)
        elif kind == "weights":
            got = oracle.weights(int(inp), int(sign))
            want = np.array(parse_complex_list(exp))
            assert np.array_equal(got, want), got  # exact: quarter turns
        elif kind == "bitrev":
            n = int(inp)
            order = [int(v) for v in exp.split()]
            assert [oracle.rev(j, n.bit_length() - 1) for j in range(n)] == order
            x = np.arange(n) + 0j
            assert np.array_equal(oracle.bitrev(x).real.astype(int), order)


def test_moa_index_example(golden_dir):
    """gamma(<3 5 4>, <2 1 3>) = 47 and <2 1> psi A = <44 45 46 47>."""
    for kind, shape, idx, want in read_golden(os.path.join(golden_dir, "moa_index.txt")):
        shape = [int(v) for v in shape.split()]
        idx = [int(v) for v in idx.split()]
        want = [int(v) for v in want.split()]
        if kind == "gamma":
            assert oracle.gamma(shape, idx) == want[0]
        else:
            got = [oracle.gamma(shape, idx + [k]) for k in range(shape[-1])]
            assert got == want
    A = np.arange(60).reshape(3, 5, 4)  # row-major items 0..59
    assert A[2, 1, 3] == 47


def test_splitmix64_reference(golden_dir):
    for line in open(os.path.join(golden_dir, "splitmix64.txt")):
        if line.startswith("#") or not line.strip():
            continue
        seed, idx, want = line.split()
        assert int(moa_inputs.splitmix64(int(seed), int(idx))) == int(want, 16)


def test_generator_range_and_moments():
    x = moa_inputs.signal_for(16)
    f = x.view(np.float64)
    assert f.min() >= -1.0 and f.max() < 1.0
    # E|x|^2 = 2/3 (SURVEY §8(d) sanity check)
    assert abs(np.mean(np.abs(x) ** 2) - 2 / 3) < 0.01
    # rank slices are the residue classes of the full signal
    for p in (2, 4, 8):
        for r in range(p):
            assert np.array_equal(moa_inputs.rank_slice(16, r, p), x[r::p])


# ---------------------------------------------------------------- weights / permutation
def test_omega_exact_quarter_turns_and_accuracy():
    for q in range(2, 21):
        L = 1 << q
        for sign in SIGNS:
            assert oracle.omega(0, L, sign) == 1
            assert oracle.omega(L // 4, L, sign) == complex(0, sign)
            assert oracle.omega(L // 2, L, sign) == -1
            assert oracle.omega(3 * L // 4, L, sign) == complex(0, -sign)
    L = 1 << 12
    e = np.arange(L)
    w = np.array([oracle.omega(int(k), L, -1) for k in e])
    ref = np.exp(-2j * np.pi * e.astype(np.longdouble) / L)  # numpy long double path
    assert np.max(np.abs(w - ref.astype(np.complex128))) < 4e-16
    assert np.max(np.abs(np.abs(w) - 1)) < 4e-16
    # conjugate symmetry between the two signs
    wp = np.array([oracle.omega(int(k), L, +1) for k in e])
    assert np.array_equal(wp, np.conj(w))


def test_weights_unit_modulus_and_powers():
    w = oracle.weights(1024, -1)
    assert w[0] == 1 and np.max(np.abs(np.abs(w) - 1)) < 1e-15
    # weight(row) = omega_L^row: successive powers of omega_L
    w1 = w[1]
    acc = np.cumprod(np.full(511, w1))
    assert np.max(np.abs(acc - w[1:])) < 1e-13


def test_bitrev_involution():
    for t in range(1, 13):
        x = _rand(1 << t, t)
        assert np.array_equal(oracle.bitrev(oracle.bitrev(x)), x)


# ---------------------------------------------------------------- DFT definition pins
@pytest.mark.parametrize("t", range(1, 11))
def test_fft_equals_bruteforce_dft(t):
    n = 1 << t
    for sign in SIGNS:
        x = moa_inputs.signal_for(t)
        assert oracle.rel_l2(oracle.fft(x, sign), oracle.dft(x, sign)) <= 1e-14


def test_dft_bins_equals_definition():
    for t in (1, 5, 10):
        x = moa_inputs.signal_for(t)
        ks = np.arange(1 << t)
        for sign in SIGNS:
            assert oracle.rel_l2(oracle.dft_bins(x, ks, sign), oracle.dft(x, sign)) <= 1e-15
    x = moa_inputs.signal_for(16)
    ks = [0, 1, 777, 40000, 65535]
    assert oracle.rel_l2(oracle.dft_bins(x, ks), np.fft.fft(x)[ks]) <= 1e-14


def test_dft_bins_range_windows_sum_to_the_definition():
    """Windows of a partition of [0, n) sum to the plain definition (numpy's FFT as the
    independent check), including a window start whose j0*k exceeds 2^63 (the 128-bit
    start exponent); a lone impulse at j0 gives omega_n^(k*j0) exactly."""
    t = 14
    n = 1 << t
    x = moa_inputs.signal_for(t)
    ks = [0, 1, 5, 4097, n // 2, n - 1]
    for sign in SIGNS:
        acc = sum(oracle.dft_bins_range(x[j0:j0 + 1024], n, j0, ks, sign) for j0 in range(0, n, 1024))
        ref = np.fft.fft(x)[ks] if sign < 0 else np.fft.ifft(x)[ks] * n
        assert oracle.rel_l2(acc, ref) <= 1e-14
    # impulse at j0 of a 2^40-point signal, bins near 2^40: (j0 * k) >> 63 != 0
    n = 1 << 40
    j0 = (1 << 40) - 3
    ks = np.array([(1 << 40) - 1, (1 << 39) + 12345, 3])
    got = oracle.dft_bins_range(np.array([1.0 + 0j]), n, j0, ks)
    want = np.exp(-2j * np.pi * ((j0 * ks) % n) / n)
    assert np.max(np.abs(got - want)) <= 1e-15


def test_dft_non_power_of_two_against_numpy():
    # the definition itself, for lengths the FFT cannot take
    for n in (1, 3, 5, 6, 7, 12, 31):
        x = _rand(n, n)
        assert oracle.rel_l2(oracle.dft(x, -1), np.fft.fft(x)) <= 1e-14
        assert oracle.rel_l2(oracle.dft(x, +1), np.fft.ifft(x) * n) <= 1e-14


@pytest.mark.parametrize("t", [1, 4, 10, 16])
def test_impulse_to_constant_bitwise(t):
    n = 1 << t
    x = np.zeros(n, complex)
    x[0] = 1
    for sign in SIGNS:
        assert np.array_equal(oracle.fft(x, sign), np.ones(n, complex))


@pytest.mark.parametrize("t", [4, 10, 16])
def test_shifted_impulse_phase_ramp(t):
    n = 1 << t
    for s in (1, 3, n // 3, n - 1):
        x = np.zeros(n, complex)
        x[s] = 1
        k = np.arange(n)
        for sign in SIGNS:
            want = np.exp(sign * 2j * np.pi * ((s * k) % n) / n)
            assert np.max(np.abs(oracle.fft(x, sign) - want)) <= 1e-14


@pytest.mark.parametrize("t", [4, 10, 16])
def test_tone_to_delta(t):
    n = 1 << t
    j = np.arange(n)
    for f in (0, 1, 5, n // 2 + 3):
        for sign in SIGNS:
            x = np.exp(-sign * 2j * np.pi * ((f * j) % n) / n)
            want = np.zeros(n, complex)
            want[f] = n
            assert np.max(np.abs(oracle.fft(x, sign) - want)) / n <= 1e-14


@pytest.mark.parametrize("t", [4, 10, 16])
def test_linearity(t):
    x = moa_inputs.signal_for(t)
    y = moa_inputs.signal_for(t, second=True)
    a, b = 0.75 - 0.5j, -1.25 + 2j
    for sign in SIGNS:
        lhs = oracle.fft(a * x + b * y, sign)
        rhs = a * oracle.fft(x, sign) + b * oracle.fft(y, sign)
        assert oracle.rel_l2(lhs, rhs) <= 1e-14


@pytest.mark.parametrize("t", [4, 10, 16, 20])
def test_parseval(t):
    x = moa_inputs.signal_for(t)
    X = oracle.fft(x, -1)
    lhs = np.sum(np.abs(X.astype(np.clongdouble)) ** 2)
    rhs = (1 << t) * np.sum(np.abs(x.astype(np.clongdouble)) ** 2)
    assert abs(lhs - rhs) / rhs <= 1e-13


@pytest.mark.parametrize("t", [4, 10, 16, 20])
def test_round_trip(t):
    x = moa_inputs.signal_for(t)
    back = oracle.fft(oracle.fft(x, -1), +1) / (1 << t)
    assert oracle.rel_l2(back, x) <= 1e-14


def test_real_input_symmetry_and_constant():
    n = 1 << 12
    x = np.random.default_rng(5).uniform(-1, 1, n) + 0j
    X = oracle.fft(x, -1)
    k = np.arange(1, n)
    assert np.max(np.abs(X[n - k] - np.conj(X[k]))) <= 1e-14 * np.max(np.abs(X))
    c = oracle.fft(np.full(n, 2.5 + 0j), -1)
    assert c[0] == 2.5 * n and np.max(np.abs(c[1:])) <= 1e-12


def test_time_shift_theorem():
    n = 1 << 10
    x = moa_inputs.signal_for(10)
    s = 37
    X = oracle.fft(x, -1)
    Xs = oracle.fft(np.roll(x, s), -1)
    k = np.arange(n)
    assert oracle.rel_l2(Xs, X * np.exp(-2j * np.pi * s * k / n)) <= 1e-14


@pytest.mark.parametrize("t", [4, 10, 16, 20])
def test_library_special_case_pocketfft(t):
    x = moa_inputs.signal_for(t)
    assert oracle.rel_l2(oracle.fft(x, -1), np.fft.fft(x)) <= 1e-14
    assert oracle.rel_l2(oracle.fft(x, +1), np.fft.ifft(x) * (1 << t)) <= 1e-14


@pytest.mark.parametrize("t", [10, 16])
def test_extended_precision_fft(t):
    x = moa_inputs.signal_for(t)
    ref = np.fft.fft(x.astype(np.clongdouble))
    assert oracle.rel_l2(oracle.fft(x, -1), ref.astype(np.complex128)) <= 2e-15


# ---------------------------------------------------------------- variants
@pytest.mark.parametrize("t", [1, 5, 12])
def test_temp_variant_bitwise(t):
    """Fig 3.8 (temp xx) and Fig 3.9 (in place) share the arithmetic order."""
    x = moa_inputs.signal_for(t)
    for sign in SIGNS:
        assert np.array_equal(oracle.fft_temp(x, sign), oracle.fft(x, sign))


def test_openmp_mode_bitwise():
    """Fig 6.1 parallel-do template: same per-element arithmetic."""
    for t in (3, 12, 18):
        x = moa_inputs.signal_for(t)
        ref = oracle.fft(x, -1, threads=1)
        for th in (2, 3, 8):
            assert np.array_equal(oracle.fft(x, -1, threads=th), ref)


# ---------------------------------------------------------------- distributed plan
@pytest.mark.parametrize("t,m", [(10, 2), (10, 4), (10, 8), (6, 8), (12, 4)])
def test_dist_sim_bitwise_all_breakpoints(t, m):
    """Fig 5.7 + Fig 5.9: equal to Fig 3.9 bitwise for every breakpoint in
    [log2 m + 1, log2 psize + 1] (§4.8); processor p ends with X[p + m*i]
    (P:799)."""
    n = 1 << t
    x = moa_inputs.signal_for(t)
    ref = oracle.fft(x, -1)
    psize = n // m
    lo, hi = int(math.log2(m)) + 1, int(math.log2(psize)) + 1
    for bp in range(lo, hi + 1):
        cyc, out, _ = oracle.dist_sim(x, m, bp, -1)
        assert np.array_equal(out, ref), bp
        for p in range(m):
            assert np.array_equal(cyc[p], ref[p::m])


def test_dist_sim_structure_counts():
    n, m = 1 << 10, 4
    psize = n // m
    x = moa_inputs.signal_for(10)
    for bp in (3, 6, 9):
        _, _, c = oracle.dist_sim(x, m, bp, -1)
        assert c["messages"] == m * (m - 1)
        assert c["elements_per_message"] == psize // m
        assert c["assigns_per_stage"] == psize
        t = 10
        assert c["weights_per_proc"] == sum((1 << q) // (2 * m) for q in range(bp, t + 1))


def test_dist_sim_rejects_bad_configs():
    x = np.zeros(16, complex)
    with pytest.raises(ValueError):
        oracle.dist_sim(x, 8)            # psize = 2 < m = 8
    x = np.zeros(64, complex)
    with pytest.raises(ValueError):
        oracle.dist_sim(x, 4, 2)         # breakpoint < log2 m + 1
    with pytest.raises(ValueError):
        oracle.dist_sim(x, 4, 6)         # breakpoint > log2 psize + 1
    for bp in (3, 4, 5):                 # n=64, m=4 -> {3,4,5}
        oracle.dist_sim(x, 4, bp)


def test_residue_class_relabeling():
    """Reading R4: the paper's processor p holds, after P_n and the block scatter,
    the residue class x[rev(p) + m*j] in bit-reversed order; the GPU's rank r owns
    x[r + P*j] in natural order."""
    t, m = 8, 4
    n = 1 << t
    x = np.arange(n) + 0j
    y = oracle.bitrev(x)
    psize = n // m
    s = int(math.log2(m))
    for p in range(m):
        block = y[p * psize:(p + 1) * psize]
        r = oracle.rev(p, s)
        assert np.array_equal(oracle.bitrev(block), x[r::m])


def test_rejects_invalid_n():
    with pytest.raises(ValueError):
        oracle.fft(np.zeros(6, complex))
    with pytest.raises(ValueError):
        oracle.fft(np.zeros(1, complex))  # t >= 1


# ------------------------------------------------------------------ 2-D via Omega (App. B)
@pytest.mark.parametrize("n1,n2", [(2, 2), (2, 8), (4, 4), (8, 2), (4, 16)])
def test_fft2_equals_bruteforce_double_sum(n1, n2):
    """fft2 (rows, transpose, rows, transpose) against the 2-D definition written out."""
    x = moa_inputs.complex_signal(0x2D2D + n1 * 131 + n2, n1 * n2).reshape(n1, n2)
    for sign in (-1, 1):
        assert oracle.rel_l2(oracle.fft2(x, sign), oracle.dft2(x, sign)) <= 1e-14


def test_fft2_separable_closed_form():
    """x = a (outer) b  =>  X = A (outer) B with A, B the 1-D transforms (closed form of
    the separable sum); a 2-D impulse goes to all ones, bitwise."""
    n1, n2 = 32, 64
    a = moa_inputs.complex_signal(11, n1)
    b = moa_inputs.complex_signal(12, n2)
    X = oracle.fft2(np.outer(a, b))
    assert oracle.rel_l2(X, np.outer(oracle.fft(a), oracle.fft(b))) <= 1e-14
    d = np.zeros((n1, n2), complex)
    d[0, 0] = 1
    assert np.array_equal(oracle.fft2(d), np.ones((n1, n2), complex))


def test_fft2_library_special_case():
    x = moa_inputs.complex_signal(0x2D, 64 * 128).reshape(64, 128)
    assert oracle.rel_l2(oracle.fft2(x, -1), np.fft.fft2(x)) <= 1e-14
    assert oracle.rel_l2(oracle.fft2(x, +1), np.fft.ifft2(x) * x.size) <= 1e-14


@pytest.mark.parametrize("shape", [(2, 2, 2), (2, 4, 8), (4, 2, 4), (8, 8)])
def test_fftn_equals_bruteforce_sum(shape):
    x = moa_inputs.complex_signal(0x3D + sum(shape), int(np.prod(shape))).reshape(shape)
    for sign in (-1, 1):
        assert oracle.rel_l2(oracle.fftn(x, sign), oracle.dftn(x, sign)) <= 1e-14


def test_fftn_matches_fft2_and_numpy():
    x = moa_inputs.complex_signal(0x3E, 16 * 32 * 8).reshape(16, 32, 8)
    assert oracle.rel_l2(oracle.fftn(x), np.fft.fftn(x)) <= 1e-14
    y = x.reshape(16, 256)
    assert np.array_equal(oracle.fftn(y), oracle.fft2(y))


def test_rel_l2_closed_forms_pin_the_checker():
    """The parity metric itself (oracle.rel_l2) against closed forms,
    so a broken checker cannot pass a wrong GPU result: one perturbed element gives
    |d| / ||x||, a swapped pair sqrt(2) |x_a - x_b| / ||x||, a scaled vector |a - 1|, a zero
    reference ||g||; and at the GPU bar (1e-12 log2 n) a perturbation of 1e-10 ||x|| fails."""
    rng = np.random.default_rng(7)
    n = 4096
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    nx = np.sqrt(np.sum(np.abs(x) ** 2))
    d = 3e-7 - 4e-7j
    y = x.copy()
    y[1234] += d
    assert abs(oracle.rel_l2(y, x) - abs(d) / nx) <= 1e-9 * abs(d) / nx
    s = x.copy()
    s[[5, 3000]] = x[[3000, 5]]
    want = np.sqrt(2) * abs(x[5] - x[3000]) / nx
    assert abs(oracle.rel_l2(s, x) - want) <= 1e-12 * want
    assert abs(oracle.rel_l2(1.5 * x, x) - 0.5) <= 1e-15
    assert oracle.rel_l2(x, x) == 0.0
    assert abs(oracle.rel_l2(x, np.zeros(n, dtype=np.complex128)) - nx) <= 1e-12 * nx
    z = x.copy()
    z[17] += 1e-10 * nx
    assert oracle.rel_l2(z, x) > 1e-12 * 12          # fails the bar at n = 2^12
    # l2_parts over chunks equals the whole sum (the chunked form the large tests use)
    a, b = oracle.l2_parts(y, x, chunk=1000)
    a2, b2 = oracle.l2_parts(y, x)
    assert abs(a - a2) <= 1e-20 and abs(b - b2) <= 1e-9
