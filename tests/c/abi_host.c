/* C99 client of include/moa_fft.h (tests/test_abi.py compiles it with gcc and runs it on
 * the CPU): the header is plain C, the library links from C, and its host-only entry
 * points answer as documented -- the default lifting of SURVEY §8 (n = 2^24 -> three
 * 256-point levels), a pass's index map, and the error codes with their messages. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "moa_fft.h"

static int fails = 0;
#define CHECK(c, ...)                          \
    do {                                       \
        if (!(c)) {                            \
            fprintf(stderr, "FAIL: " __VA_ARGS__); \
            fprintf(stderr, "\n");             \
            ++fails;                           \
        }                                      \
    } while (0)

int main(void) {
    int64_t lift[4];
    int d = 0;
    CHECK(moa_fft_default_lifting((int64_t)1 << 24, 1, lift, &d) == MOA_OK, "default_lifting");
    CHECK(d == 3 && lift[0] == 256 && lift[1] == 256 && lift[2] == 256, "lifting of 2^24 = <256,256,256>");
    CHECK(moa_fft_default_lifting(6, 1, lift, &d) == MOA_ERR_INVALID_N, "n = 6 rejected");
    CHECK(moa_fft_last_error_code() == MOA_ERR_INVALID_N, "last_error_code INVALID_N");
    CHECK(strstr(moa_fft_last_error(), "2^t") != NULL, "message names the bound: %s", moa_fft_last_error());
    CHECK(moa_fft_default_lifting(16, 8, lift, &d) == MOA_ERR_INVALID_P, "psize < m rejected (P:289)");
    /* pass 0 of n = 64 = <8, 8>: column DFTs over stride 8, in place, twiddle omega_64^(b k) */
    const int64_t n = 64;
    int64_t *in = malloc(n * sizeof *in), *out = malloc(n * sizeof *out), *tw = malloc(n * sizeof *tw), F = 0;
    moa_fft_options o;
    memset(&o, 0, sizeof o);
    o.nlift = 2;
    o.lift[0] = 8;
    o.lift[1] = 8;
    CHECK(moa_fft_describe_pass(n, 1, 0, &o, 0, in, out, tw, &F) == MOA_OK, "describe_pass");
    CHECK(F == 8, "F = 8");
    int covered[64] = {0};
    for (int64_t i = 0; i < n; ++i) {
        CHECK(in[i] >= 0 && in[i] < n, "index in range");
        covered[in[i]] += 1;
        CHECK(in[i] % 8 == in[i - i % 8] % 8, "one transform = one column (stride 8)");
        CHECK(out[i] == in[i], "middle pass stores in place");
        CHECK(tw[i] == ((in[i] % 8) * (in[i] / 8)) % 64, "twiddle omega_64^(b k): b = column, k = point");
    }
    for (int i = 0; i < 64; ++i) CHECK(covered[i] == 1, "every element once");
    printf("%s %s\n", fails ? "FAILED" : "OK", moa_fft_version());
    free(in);
    free(out);
    free(tw);
    return fails ? 1 : 0;
}
