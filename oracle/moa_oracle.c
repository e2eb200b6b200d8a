/*
 * moa_oracle.c -- the CPU ORACLE for the MoA reshape-transpose FFT.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is never part of the product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load or call it.  It shares no code, header, table or
 * constant generator with paper_0811_2535_b200/ (the CUDA path), and neither
 * side includes or imports the other.
 *
 * It is deliberately plain and slow: every function follows one figure of
 *   Hunt, Mullin, Rosenkrantz, Raynolds, "A transformation-based approach for
 *   the design of parallel/distributed scientific software: the FFT"
 *   (arXiv 0811.2535), cited as P:<line of /root/reference/PAPER.md>.
 * in the paper's order and notation (x, xx, q, L, row, col', weight, psize,
 * breakpoint, xblock, xcyclic, weightcyclic, myid/p, m).
 *
 * Conventions:
 *   - complex numbers are interleaved (re, im) doubles;
 *   - sign in {-1,+1}: weight(row) = exp(sign * 2*pi*i*row/L).  The paper's
 *     code literally writes EXP((2*pi*i*row)/L) = sign +1; sign -1 is
 *     the conventional forward DFT (reading R1);
 *   - no normalisation in either direction (reading R2);
 *   - the complex product is (ac - bd, ad + bc), compiled with
 *     -ffp-contract=off so there is no FMA (reading R12): the result is
 *     deterministic and the multi-threaded mode is bitwise equal to 1 thread.
 *
 * Pins (tests/test_oracle.py): brute-force DFT for n <= 2^10, the SPEC
 * worked values, impulse/tone closed forms, linearity, Parseval, round trip,
 * real-input symmetry, numpy.fft (pocketfft) and the extended-precision
 * clongdouble FFT, and the distributed layout X[p + m*i].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_EINVAL (-1)
#define ORACLE_ENOMEM (-2)

/* n = 2^t with t >= 1 (Fig 2.1 input).  Returns t or -1. */
static int log2_exact(int64_t n) {
    if (n < 1 || (n & (n - 1)) != 0) return -1;
    int t = 0;
    while (((int64_t)1 << t) < n) ++t;
    return t;
}

/* rev_t(j): reverse the t-bit binary representation of j. */
int64_t oracle_rev(int64_t j, int t) {
    int64_t r = 0;
    for (int b = 0; b < t; ++b) {
        r = (r << 1) | (j & 1);
        j >>= 1;
    }
    return r;
}

/*
 * exp(sign * 2*pi*i * e / L) for integer e, L = 2^q (the paper's weight,
 * Fig 3.8 "weight(row) = EXP((2*pi*i*row)/L)").
 * Evaluated in long double after reducing e/L to the first octant, so the
 * quarter turns e/L in {0, 1/4, 1/2, 3/4} are exact (1, i, -1, -i) and the
 * rest is the correctly-rounded-to-double value of a long-double cos/sin.
 */
void oracle_omega(int64_t e, int64_t L, int sign, double out[2]) {
    const long double half_pi = 1.5707963267948966192313216916397514L;
    e %= L;
    if (e < 0) e += L;
    /* theta = 2*pi*e/L = (pi/2) * (qd + r/L), qd = quadrant */
    int64_t qd = (4 * e) / L;
    int64_t r = (4 * e) % L;           /* 0 <= r < L, angle within quadrant = (pi/2) r/L */
    long double c, s;
    if (r == 0) {
        c = 1.0L;
        s = 0.0L;
    } else if (2 * r <= L) {           /* phi = (pi/2) r/L <= pi/4 */
        long double phi = half_pi * (long double)r / (long double)L;
        c = cosl(phi);
        s = sinl(phi);
    } else {                           /* phi > pi/4: use the complementary angle */
        long double psi = half_pi * (long double)(L - r) / (long double)L;
        c = sinl(psi);
        s = cosl(psi);
    }
    long double re, im;
    switch (qd) {                      /* rotate by qd quarter turns */
    case 0: re = c; im = s; break;
    case 1: re = -s; im = c; break;
    case 2: re = -c; im = -s; break;
    default: re = s; im = -c; break;
    }
    out[0] = (double)re;
    out[1] = (double)(sign < 0 ? -im : im);
}

/* Line 1 of Fig 2.1: x <- P_n x, y[j] = x[rev_t(j)]. */
int oracle_bitrev(int64_t n, const double *x, double *y) {
    int t = log2_exact(n);
    if (t < 0) return ORACLE_EINVAL;
    for (int64_t j = 0; j < n; ++j) {
        int64_t r = oracle_rev(j, t);
        y[2 * j] = x[2 * r];
        y[2 * j + 1] = x[2 * r + 1];
    }
    return ORACLE_OK;
}

/* weight(row) = EXP(sign*2*pi*i*row/L), row = 0..L/2-1 (Fig 3.8). */
int oracle_weights(int64_t L, int sign, double *weight) {
    if (log2_exact(L) < 1) return ORACLE_EINVAL;
    for (int64_t row = 0; row < L / 2; ++row) oracle_omega(row, L, sign, &weight[2 * row]);
    return ORACLE_OK;
}

/*
 * Fig 3.7 basic block: c = weight(row)*x(col'+row+L/2); d = x(col'+row);
 * x(col'+row) = d + c; x(col'+row+L/2) = d - c.
 */
static inline void basic_block(double *x, int64_t lo, int64_t hi, const double *w) {
    double ar = w[0], ai = w[1];
    double br = x[2 * hi], bi = x[2 * hi + 1];
    double cr = ar * br - ai * bi;
    double ci = ar * bi + ai * br;
    double dr = x[2 * lo], di = x[2 * lo + 1];
    x[2 * lo] = dr + cr;
    x[2 * lo + 1] = di + ci;
    x[2 * hi] = dr - cr;
    x[2 * hi + 1] = di - ci;
}

/*
 * Fig 3.9 "Loop with In-Place Butterfly Computation", run on a
 * vector that has already been bit-reversed (Fig 2.1 line 1).
 * threads > 1 selects the Fig 6.1 all-processor template: the
 * col' loop (or, once there are fewer columns than threads, the row loop) is
 * a `parallel do`; every element sees the same arithmetic, so the result is
 * bitwise identical to threads == 1.
 */
static int fft_stages(int64_t n, int t, int sign, int threads, double *x) {
    double *weight = (double *)malloc(sizeof(double) * (size_t)(n > 1 ? n : 2));
    if (!weight) return ORACLE_ENOMEM;
    (void)threads;
    for (int q = 1; q <= t; ++q) {
        int64_t L = (int64_t)1 << q;
        for (int64_t row = 0; row <= L / 2 - 1; ++row) oracle_omega(row, L, sign, &weight[2 * row]);
        int64_t ncols = n / L;
#ifdef _OPENMP
        if (threads > 1 && ncols >= threads) {
#pragma omp parallel for num_threads(threads) schedule(static)
            for (int64_t col = 0; col < ncols; ++col) {
                int64_t colp = col * L;
                for (int64_t row = 0; row <= L / 2 - 1; ++row)
                    basic_block(x, colp + row, colp + row + L / 2, &weight[2 * row]);
            }
            continue;
        }
        if (threads > 1) {
            for (int64_t colp = 0; colp <= n - 1; colp += L) {
#pragma omp parallel for num_threads(threads) schedule(static)
                for (int64_t row = 0; row <= L / 2 - 1; ++row)
                    basic_block(x, colp + row, colp + row + L / 2, &weight[2 * row]);
            }
            continue;
        }
#endif
        for (int64_t colp = 0; colp <= n - 1; colp += L)        /* do col' = 0,n-1,L */
            for (int64_t row = 0; row <= L / 2 - 1; ++row)      /*   do row = 0,L/2-1 */
                basic_block(x, colp + row, colp + row + L / 2, &weight[2 * row]);
    }
    free(weight);
    return ORACLE_OK;
}

/*
 * The oracle FFT: Fig 2.1 literally in the Fig 3.9 in-place form.
 * X_k = sum_j x_j exp(sign*2*pi*i*j*k/n), no normalisation.  in may equal out.
 */
int oracle_fft(int64_t n, int sign, int threads, const double *in, double *out) {
    int t = log2_exact(n);
    if (t < 1 || (sign != 1 && sign != -1)) return ORACLE_EINVAL;
    double *y = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    if (!y) return ORACLE_ENOMEM;
    oracle_bitrev(n, in, y);                          /* (1) x <- P_n x */
    int rc = fft_stages(n, t, sign, threads, y);      /* (2)-(7) */
    if (rc == ORACLE_OK) memcpy(out, y, sizeof(double) * 2 * (size_t)n);
    free(y);
    return rc;
}

/*
 * Fig 3.8 "Loop with Optimized Basic Block": the same stages with
 * the temporary xx and the copy x = xx.  Must equal Fig 3.9 bitwise (P:243:
 * the in-place form only replaces xx by the scalar d).
 */
int oracle_fft_temp(int64_t n, int sign, const double *in, double *out) {
    int t = log2_exact(n);
    if (t < 1 || (sign != 1 && sign != -1)) return ORACLE_EINVAL;
    double *x = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    double *xx = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    double *weight = (double *)malloc(sizeof(double) * (size_t)n);
    if (!x || !xx || !weight) {
        free(x); free(xx); free(weight);
        return ORACLE_ENOMEM;
    }
    oracle_bitrev(n, in, x);
    for (int q = 1; q <= t; ++q) {
        int64_t L = (int64_t)1 << q;
        for (int64_t row = 0; row <= L / 2 - 1; ++row) oracle_omega(row, L, sign, &weight[2 * row]);
        for (int64_t colp = 0; colp <= n - 1; colp += L) {
            for (int64_t row = 0; row <= L / 2 - 1; ++row) {
                int64_t lo = colp + row, hi = colp + row + L / 2;
                double ar = weight[2 * row], ai = weight[2 * row + 1];
                double cr = ar * x[2 * hi] - ai * x[2 * hi + 1];
                double ci = ar * x[2 * hi + 1] + ai * x[2 * hi];
                xx[2 * lo] = x[2 * lo] + cr;
                xx[2 * lo + 1] = x[2 * lo + 1] + ci;
                xx[2 * hi] = x[2 * lo] - cr;
                xx[2 * hi + 1] = x[2 * lo + 1] - ci;
            }
        }
        memcpy(x, xx, sizeof(double) * 2 * (size_t)n);  /* x = xx */
    }
    memcpy(out, x, sizeof(double) * 2 * (size_t)n);
    free(x); free(xx); free(weight);
    return ORACLE_OK;
}

/*
 * The plain definition the FFT reaches: X_k = sum_{j ascending} x_j * W[(j*k) mod n],
 * W[e] = exp(sign*2*pi*i*e/n), accumulated in long double.  O(n^2): small n only.
 * Any n >= 1 (not only powers of two) -- the definition does not need 2^t.
 */
int oracle_dft(int64_t n, int sign, const double *in, double *out) {
    if (n < 1 || (sign != 1 && sign != -1)) return ORACLE_EINVAL;
    long double *W = (long double *)malloc(sizeof(long double) * 2 * (size_t)n);
    if (!W) return ORACLE_ENOMEM;
    const long double two_pi = 6.2831853071795864769252867665590058L;
    for (int64_t e = 0; e < n; ++e) {
        long double a = two_pi * (long double)e / (long double)n;
        W[2 * e] = cosl(a);
        W[2 * e + 1] = (sign < 0 ? -1.0L : 1.0L) * sinl(a);
    }
    for (int64_t k = 0; k < n; ++k) {
        long double sr = 0.0L, si = 0.0L;
        for (int64_t j = 0; j < n; ++j) {
            int64_t e = (int64_t)(((unsigned __int128)j * (unsigned __int128)k) % (unsigned __int128)n);
            long double xr = in[2 * j], xi = in[2 * j + 1];
            sr += xr * W[2 * e] - xi * W[2 * e + 1];
            si += xr * W[2 * e + 1] + xi * W[2 * e];
        }
        out[2 * k] = (double)sr;
        out[2 * k + 1] = (double)si;
    }
    free(W);
    return ORACLE_OK;
}

/*
 * The same definition evaluated at selected bins only (for sampled parity at
 * sizes where the O(n log n) oracle does not fit in host memory/time):
 * X_k = sum_{j ascending} x_j w^{jk mod n}, long double accumulation, with
 * w^e = W_hi[e >> h] * W_lo[e & (2^h - 1)] built in long double per call.
 * n must be a power of two (the split needs it); any k in [0, n).
 */
int oracle_dft_bins(int64_t n, int sign, const double *in, int64_t nk, const int64_t *ks, double *out) {
    int t = log2_exact(n);
    if (t < 0 || (sign != 1 && sign != -1)) return ORACLE_EINVAL;
    int h = (t + 1) / 2;
    int64_t nlo = (int64_t)1 << h, nhi = n >> h;
    long double *Wlo = (long double *)malloc(sizeof(long double) * 2 * (size_t)nlo);
    long double *Whi = (long double *)malloc(sizeof(long double) * 2 * (size_t)nhi);
    if (!Wlo || !Whi) {
        free(Wlo); free(Whi);
        return ORACLE_ENOMEM;
    }
    const long double two_pi = 6.2831853071795864769252867665590058L;
    const long double sg = sign < 0 ? -1.0L : 1.0L;
    for (int64_t e = 0; e < nlo; ++e) {
        long double a = two_pi * (long double)e / (long double)n;
        Wlo[2 * e] = cosl(a);
        Wlo[2 * e + 1] = sg * sinl(a);
    }
    for (int64_t e = 0; e < nhi; ++e) {
        long double a = two_pi * (long double)(e << h) / (long double)n;
        Whi[2 * e] = cosl(a);
        Whi[2 * e + 1] = sg * sinl(a);
    }
    for (int64_t b = 0; b < nk; ++b) {
        int64_t k = ks[b] & (n - 1);
        long double sr = 0.0L, si = 0.0L;
        uint64_t e = 0;                       /* j*k mod n, updated incrementally */
        for (int64_t j = 0; j < n; ++j) {
            const long double *wl = &Wlo[2 * (e & (uint64_t)(nlo - 1))];
            const long double *wh = &Whi[2 * (e >> h)];
            long double wr = wh[0] * wl[0] - wh[1] * wl[1];
            long double wi = wh[0] * wl[1] + wh[1] * wl[0];
            long double xr = in[2 * j], xi = in[2 * j + 1];
            sr += xr * wr - xi * wi;
            si += xr * wi + xi * wr;
            e = (e + (uint64_t)k) & (uint64_t)(n - 1);
        }
        out[2 * b] = (double)sr;
        out[2 * b + 1] = (double)si;
    }
    free(Wlo); free(Whi);
    return ORACLE_OK;
}

/*
 * The plain definition restricted to a window of the input:
 *   out_b = sum_{j=0}^{len-1} x[j0 + j] * omega_n^(sign * k_b * (j0 + j)),
 * with in = x + j0 (len elements).  Summing the windows of a partition of [0, n)
 * gives dft_bins; it lets a test stream an input too large for host memory.
 */
int oracle_dft_bins_range(int64_t n, int sign, const double *in, int64_t j0, int64_t len, int64_t nk,
                          const int64_t *ks, double *out) {
    int t = log2_exact(n);
    if (t < 0 || (sign != 1 && sign != -1) || j0 < 0 || len < 0 || j0 + len > n) return ORACLE_EINVAL;
    int h = (t + 1) / 2;
    int64_t nlo = (int64_t)1 << h, nhi = n >> h;
    long double *Wlo = (long double *)malloc(sizeof(long double) * 2 * (size_t)nlo);
    long double *Whi = (long double *)malloc(sizeof(long double) * 2 * (size_t)nhi);
    if (!Wlo || !Whi) {
        free(Wlo); free(Whi);
        return ORACLE_ENOMEM;
    }
    const long double two_pi = 6.2831853071795864769252867665590058L;
    const long double sg = sign < 0 ? -1.0L : 1.0L;
    for (int64_t e = 0; e < nlo; ++e) {
        long double a = two_pi * (long double)e / (long double)n;
        Wlo[2 * e] = cosl(a);
        Wlo[2 * e + 1] = sg * sinl(a);
    }
    for (int64_t e = 0; e < nhi; ++e) {
        long double a = two_pi * (long double)(e << h) / (long double)n;
        Whi[2 * e] = cosl(a);
        Whi[2 * e + 1] = sg * sinl(a);
    }
    for (int64_t b = 0; b < nk; ++b) {
        int64_t k = ks[b] & (n - 1);
        long double sr = 0.0L, si = 0.0L;
        /* (j0 + j)*k mod n, updated incrementally (128-bit start: j0*k can exceed 2^63) */
        uint64_t e = (uint64_t)(((unsigned __int128)(uint64_t)j0 * (uint64_t)k) & (unsigned __int128)(n - 1));
        for (int64_t j = 0; j < len; ++j) {
            const long double *wl = &Wlo[2 * (e & (uint64_t)(nlo - 1))];
            const long double *wh = &Whi[2 * (e >> h)];
            long double wr = wh[0] * wl[0] - wh[1] * wl[1];
            long double wi = wh[0] * wl[1] + wh[1] * wl[0];
            long double xr = in[2 * j], xi = in[2 * j + 1];
            sr += xr * wr - xi * wi;
            si += xr * wi + xi * wr;
            e = (e + (uint64_t)k) & (uint64_t)(n - 1);
        }
        out[2 * b] = (double)sr;
        out[2 * b + 1] = (double)si;
    }
    free(Wlo); free(Whi);
    return ORACLE_OK;
}

/*
 * Fig 5.7 per-processor template with partitioned data, with the
 * direct block-partitioned -> cyclic-partitioned redistribution of Fig 5.9
 * (P:1047-1062), simulated for m virtual processors run one after another.
 *
 *   proc 0 : x0 = P_n x                         (Fig 2.1 line 1; placement, reading R4)
 *   all p  : xblock_p = x0(p*psize : (p+1)*psize-1)        (Fig 5.8)
 *   all p  : q = 1..breakpoint-1 block loop on xblock_p    (Fig 5.7)
 *   all p  : xcyclic_p(otherp*psize/m + i) = xblock_otherp(p + m*i)
 *                                                          (Fig 5.9)
 *   all p  : q = breakpoint..t cyclic loop with weightcyclic(row') =
 *            EXP(sign*2*pi*i*(m*row'+p)/L)                  (Fig 5.7)
 *   gather : x0(p : n-1 : m) = xcyclic_p                    (Fig 5.8)
 *
 * out_cyclic (m*psize complex) receives xcyclic_0, xcyclic_1, ... back to back
 * (processor p's final local array), out (n complex, may be NULL) the gather.
 * breakpoint must satisfy log2(m)+1 <= breakpoint <= log2(psize)+1 (§4.8)
 * and psize >= m.  counts (may be NULL) receives
 *   [0] messages sent in the redistribution (m(m-1))
 *   [1] elements each processor sends per message (psize/m)
 *   [2] weights computed per processor over the whole cyclic loop (sum L/(2m))
 *   [3] butterfly assignments per processor per cyclic stage (psize)
 */
int oracle_dist_sim(int64_t n, int m, int breakpoint, int sign, const double *x,
                    double *out_cyclic, double *out, int64_t *counts) {
    int t = log2_exact(n);
    int lm = log2_exact(m);
    if (t < 1 || lm < 0 || (sign != 1 && sign != -1)) return ORACLE_EINVAL;
    int64_t psize = n / m;
    if (psize < m) return ORACLE_EINVAL;
    int lps = log2_exact(psize);
    if (breakpoint < lm + 1 || breakpoint > lps + 1) return ORACLE_EINVAL;

    double *x0 = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    double *xblock = (double *)malloc(sizeof(double) * 2 * (size_t)n);   /* m local arrays */
    double *xcyclic = (double *)malloc(sizeof(double) * 2 * (size_t)n);  /* m local arrays */
    double *weight = (double *)malloc(sizeof(double) * (size_t)n + 16);
    if (!x0 || !xblock || !xcyclic || !weight) {
        free(x0); free(xblock); free(xcyclic); free(weight);
        return ORACLE_ENOMEM;
    }
    oracle_bitrev(n, x, x0);

    int64_t msgs = 0, weights_computed = 0, assigns_per_stage = -1;
    for (int myid = 0; myid < m; ++myid) {
        double *xb = xblock + 2 * (size_t)myid * (size_t)psize;
        /* DISTRIBUTE_CENTRALIZED_TO_BLOCK_PARTITIONED */
        memcpy(xb, x0 + 2 * (size_t)myid * (size_t)psize, sizeof(double) * 2 * (size_t)psize);
        for (int q = 1; q <= breakpoint - 1; ++q) {
            int64_t L = (int64_t)1 << q;
            for (int64_t row = 0; row <= L / 2 - 1; ++row) oracle_omega(row, L, sign, &weight[2 * row]);
            for (int64_t colpp = 0; colpp <= psize - 1; colpp += L)
                for (int64_t row = 0; row <= L / 2 - 1; ++row)
                    basic_block(xb, colpp + row, colpp + row + L / 2, &weight[2 * row]);
        }
    }
    /* DISTRIBUTE_BLOCK_PARTITIONED_TO_CYCLIC_PARTITIONED (Fig 5.9) */
    int64_t chunk = psize / m;
    for (int myid = 0; myid < m; ++myid) {
        double *xc = xcyclic + 2 * (size_t)myid * (size_t)psize;
        for (int otherp = 0; otherp < m; ++otherp) {
            const double *xb_other = xblock + 2 * (size_t)otherp * (size_t)psize;
            /* self: xcyclic(myid*psize/m : ...) = xblock(myid:psize-1:m);
               other: RECEIVE(xcyclic(otherp*psize/m), psize/m, otherp) of
                      SEND(xblock_otherp(myid:psize-1:m), psize/m, myid) */
            for (int64_t i = 0; i < chunk; ++i) {
                xc[2 * (otherp * chunk + i)] = xb_other[2 * (myid + (int64_t)m * i)];
                xc[2 * (otherp * chunk + i) + 1] = xb_other[2 * (myid + (int64_t)m * i) + 1];
            }
            if (otherp != myid) ++msgs;
        }
    }
    for (int myid = 0; myid < m; ++myid) {
        double *xc = xcyclic + 2 * (size_t)myid * (size_t)psize;
        int64_t assigns = 0;
        for (int q = breakpoint; q <= t; ++q) {
            int64_t L = (int64_t)1 << q;
            int64_t half = L / (2 * m);
            for (int64_t rowp = 0; rowp <= half - 1; ++rowp) {
                oracle_omega((int64_t)m * rowp + myid, L, sign, &weight[2 * rowp]);
                if (myid == 0) ++weights_computed;
            }
            assigns = 0;
            for (int64_t colpp = 0; colpp <= psize - 1; colpp += L / m)
                for (int64_t rowp = 0; rowp <= half - 1; ++rowp) {
                    basic_block(xc, colpp + rowp, colpp + rowp + half, &weight[2 * rowp]);
                    assigns += 2;
                }
        }
        if (breakpoint <= t) {
            if (assigns_per_stage < 0) assigns_per_stage = assigns;
            else if (assigns_per_stage != assigns) assigns_per_stage = -2;
        }
    }
    memcpy(out_cyclic, xcyclic, sizeof(double) * 2 * (size_t)n);
    if (out) {
        /* DISTRIBUTE_CYCLIC_PARTITIONED_TO_CENTRALIZED: x0(p:n-1:m) = xcyclic_p */
        for (int p = 0; p < m; ++p)
            for (int64_t i = 0; i < psize; ++i) {
                out[2 * (p + (int64_t)m * i)] = xcyclic[2 * ((int64_t)p * psize + i)];
                out[2 * (p + (int64_t)m * i) + 1] = xcyclic[2 * ((int64_t)p * psize + i) + 1];
            }
    }
    if (counts) {
        counts[0] = msgs;
        counts[1] = chunk;
        counts[2] = weights_computed;
        counts[3] = assigns_per_stage;
    }
    free(x0); free(xblock); free(xcyclic); free(weight);
    return ORACLE_OK;
}

/*
 * Row-major gamma offset of Def A.1: x_0 = i_0, x_j = x_{j-1}*s_j + i_j.
 * Used by the plan-simulation tests; pinned by gamma(<3 5 4>, <2 1 3>) = 47.
 */
int64_t oracle_gamma(int d, const int64_t *shape, const int64_t *index) {
    int64_t off = 0;
    for (int j = 0; j < d; ++j) off = off * shape[j] + index[j];
    return off;
}

/* Threads the OpenMP mode can use (1 when built without OpenMP). */
int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
